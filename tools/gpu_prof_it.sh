mkdir -p gpurun_out
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_row -s 6 -c 2 -o gpurun_out/it_full -f python tools/prof_smooth.py > gpurun_out/ncu_it.log 2>&1
true
