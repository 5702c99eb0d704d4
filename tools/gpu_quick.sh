# quick GPU check: parity tests + e2e probe + short bench (with e2e)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
timeout 600 python bench.py --steps 50 --no-cpu --no-cufft > gpurun_out/bench_quick.log 2>&1
true
