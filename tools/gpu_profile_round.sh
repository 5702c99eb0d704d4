# Round profile: smoke, bench (all legs), reference arm, ncu launch list of the bench,
# ncu --set full of one frame's pass sequence at 1080p (warm L2, as in the real
# sequence) and at 4K, summarised on the box (gpurun_out/ must stay < 64 MiB)
mkdir -p gpurun_out/prof
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cufft --no-c4 --no-c5 --no-dropin --no-gray > gpurun_out/ncu_launch.log 2>&1
timeout 1200 ncu --set full --cache-control none --clock-control none --import-source on -k regex:'k_row|k_col' -s 27 -c 9 -o gpurun_out/seq_full -f python tools/prof_smooth.py > gpurun_out/ncu_seq.log 2>&1
timeout 1200 ncu --set full --cache-control none --clock-control none -k regex:'k_row|k_col' -s 9 -c 9 -o /tmp/seq_4k -f python tools/prof_smooth.py --frames 2 --h 2160 --w 3840 > gpurun_out/ncu_seq4k.log 2>&1
python tools/ncu_summary.py gpurun_out/seq_full.ncu-rep gpurun_out/prof/seq_full_summary.txt > /dev/null 2>&1
python tools/ncu_summary.py /tmp/seq_4k.ncu-rep gpurun_out/prof/seq_4k_summary.txt "one 4K RGB frame" traffic_4k.json > /dev/null 2>&1
true
