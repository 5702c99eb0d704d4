: > gpurun_out/roll_sweep.log
for e in "ILS_X=0" "ILS_ROLL_ROWS=12" "ILS_ROLL_ROWS=16" "ILS_ROLL_ROWS=30" "ILS_ROLL_ROWS=45" "ILS_ROLL_PF=1"; do
  echo "== [$e]" >> gpurun_out/roll_sweep.log
  env $e timeout 300 python tools/time_passes.py --h 2160 --w 3840 | grep -o '"row_f0.*' >> gpurun_out/roll_sweep.log 2>&1
  env $e timeout 300 python tools/time_passes.py --h 4320 --w 7680 --reps 10 | grep -o '"row_f0.*' >> gpurun_out/roll_sweep.log 2>&1
done
cat gpurun_out/roll_sweep.log
