mkdir -p gpurun_out
: > gpurun_out/c45q.log
timeout 900 python -m pytest tests -m gpu -x -q >> gpurun_out/c45q.log 2>&1
timeout 300 python tools/time_passes.py --h 2160 --w 3840 --reps 20 >> gpurun_out/c45q.log 2>&1
timeout 300 python tools/time_passes.py --h 4320 --w 7680 --reps 10 >> gpurun_out/c45q.log 2>&1
timeout 600 python tools/bench_c4.py >> gpurun_out/c45q.log 2>&1
timeout 600 python tools/bench_c5.py --steps 20 >> gpurun_out/c45q.log 2>&1
timeout 600 python tools/bench_c5.py --slab --check --steps 10 >> gpurun_out/c45q.log 2>&1
true
