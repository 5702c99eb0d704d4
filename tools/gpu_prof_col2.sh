mkdir -p gpurun_out
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_col2 -s 8 -c 1 -o gpurun_out/col2_full -f python tools/prof_smooth.py > gpurun_out/ncu_col2.log 2>&1
true
