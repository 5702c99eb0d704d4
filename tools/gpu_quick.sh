# quick GPU check: parity tests + pass timings + instruction counts + short bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/time_passes.py > gpurun_out/passes.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --cache-control none --clock-control none -k regex:'k_row|k_col' -c 12 --csv --log-file gpurun_out/quick_inst.csv python tools/prof_passes.py --reps 3 > /dev/null 2>&1
timeout 600 python bench.py --steps 50 --no-cpu --no-cufft > gpurun_out/bench_quick.log 2>&1
true
