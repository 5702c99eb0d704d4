mkdir -p gpurun_out
: > gpurun_out/c4sweep.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "4k or slab or c5" >> gpurun_out/c4sweep.log 2>&1
for s in 7 8 9; do echo "spec $s" >> gpurun_out/c4sweep.log; ILS_COL2_SPEC=$s timeout 300 python tools/bench_c4.py >> gpurun_out/c4sweep.log 2>&1; done
echo "no col2" >> gpurun_out/c4sweep.log; ILS_NO_COL2=1 timeout 300 python tools/bench_c4.py >> gpurun_out/c4sweep.log 2>&1
true
