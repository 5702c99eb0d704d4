mkdir -p gpurun_out
: > gpurun_out/c5check.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pipeline or slab" >> gpurun_out/c5check.log 2>&1
timeout 600 python tools/bench_c5.py --slab --check --steps 10 >> gpurun_out/c5check.log 2>&1
timeout 600 python tools/bench_c5.py --slab --check --steps 10 --no-overlap >> gpurun_out/c5check.log 2>&1
true
