mkdir -p gpurun_out
: > gpurun_out/c5sweep.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "4k or slab or c5" >> gpurun_out/c5sweep.log 2>&1
timeout 300 python tools/bench_c5.py >> gpurun_out/c5sweep.log 2>&1
timeout 300 python tools/bench_c5.py --slab --check >> gpurun_out/c5sweep.log 2>&1
echo "no col2" >> gpurun_out/c5sweep.log; ILS_NO_COL2=1 timeout 300 python tools/bench_c5.py >> gpurun_out/c5sweep.log 2>&1
timeout 300 python tools/bench_c4.py >> gpurun_out/c5sweep.log 2>&1
true
