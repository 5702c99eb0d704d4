# quick GPU check: parity tests + pass timings (new vs old column kernel) + short bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/time_passes.py > gpurun_out/passes.log 2>&1
ILS_NO_COL2=1 timeout 300 python tools/time_passes.py >> gpurun_out/passes.log 2>&1
timeout 600 python bench.py --steps 50 --no-cpu --no-cufft --no-e2e > gpurun_out/bench_quick.log 2>&1
ILS_NO_COL2=1 timeout 600 python bench.py --steps 50 --no-cpu --no-cufft --no-e2e >> gpurun_out/bench_quick.log 2>&1
true
