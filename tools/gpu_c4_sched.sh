mkdir -p gpurun_out
: > gpurun_out/c4sched.log
timeout 300 python tools/time_passes.py --h 2160 --w 3840 >> gpurun_out/c4sched.log 2>&1
timeout 300 python tools/time_passes.py --h 4320 --w 7680 --reps 10 >> gpurun_out/c4sched.log 2>&1
timeout 300 python tools/time_passes.py --h 2160 --w 3840 --planes 1 >> gpurun_out/c4sched.log 2>&1
timeout 600 python tools/c4_planes.py >> gpurun_out/c4sched.log 2>&1
timeout 600 python -m pytest tests/test_gpu_rowroll.py -q -p no:cacheprovider >> gpurun_out/c4sched.log 2>&1
true
