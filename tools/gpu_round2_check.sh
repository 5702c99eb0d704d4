# round-2 GPU check: all GPU tests, pass timings at 1080p / 4K / 8K, the full bench line
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/passes.log
timeout 300 python tools/time_passes.py >> gpurun_out/passes.log 2>&1
timeout 300 python tools/time_passes.py --h 2160 --w 3840 >> gpurun_out/passes.log 2>&1
timeout 300 python tools/time_passes.py --h 4320 --w 7680 --reps 10 >> gpurun_out/passes.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
true
