set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cufft > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_row -s 20 -c 2 -o gpurun_out/row_full -f python tools/prof_smooth.py > gpurun_out/ncu_row.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_col -s 20 -c 1 -o gpurun_out/col_full -f python tools/prof_smooth.py > gpurun_out/ncu_col.log 2>&1
true
