# quick GPU check: parity tests + pass timings + instruction counts + e2e probe + short bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/time_passes.py > gpurun_out/passes.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --cache-control none --clock-control none -k regex:'k_row|k_col|k_u8' -c 12 --csv --log-file gpurun_out/quick_inst.csv python tools/time_u8.py --frames 1 > /dev/null 2>&1
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
timeout 600 python bench.py --steps 50 --no-cpu --no-cufft > gpurun_out/bench_quick.log 2>&1
true
