# rolling row pass vs k_row at 4K / 8K: bitwise diagnostics, pass timings (prefetch depth 0 / 1)
mkdir -p gpurun_out
timeout 600 python tools/roll_diag.py > gpurun_out/roll_diag.log 2>&1
: > gpurun_out/passes.log
for cfg in "ILS_NO_ROLL=1" "ILS_ROLL_PF=0" "ILS_ROLL_PF=1"; do
  env $cfg timeout 300 python tools/time_passes.py --h 2160 --w 3840 >> gpurun_out/passes.log 2>&1
  env $cfg timeout 300 python tools/time_passes.py --h 4320 --w 7680 --reps 10 >> gpurun_out/passes.log 2>&1
done
true
