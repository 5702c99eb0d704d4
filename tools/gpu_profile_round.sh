# Round profile: bench (all legs), reference arm, ncu launch list of the bench,
# ncu --set full of one frame's pass sequence (warm L2, as in the real sequence).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cufft > gpurun_out/ncu_launch.log 2>&1
timeout 1200 ncu --set full --cache-control none --clock-control none --import-source on -k regex:'k_row|k_col2' -s 27 -c 9 -o gpurun_out/seq_full -f python tools/prof_smooth.py > gpurun_out/ncu_seq.log 2>&1
true
timeout 600 python tools/bench_c4.py > gpurun_out/c4.log 2>&1
timeout 600 python tools/bench_c5.py --steps 10 > gpurun_out/c5.log 2>&1
timeout 600 python tools/bench_c5.py --slab --check --steps 10 >> gpurun_out/c5.log 2>&1
