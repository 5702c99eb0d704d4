mkdir -p gpurun_out
: > gpurun_out/c4band.log
for b in 0 4 3 2; do
  echo "== band $b" >> gpurun_out/c4band.log
  if [ "$b" = 0 ]; then B=""; else B=$b; fi
  ILS_ROW_BAND=$B timeout 300 python tools/time_passes.py --h 2160 --w 3840 --reps 20 >> gpurun_out/c4band.log 2>&1
  ILS_ROW_BAND=$B timeout 300 python tools/bench_c4.py --frames 128 >> gpurun_out/c4band.log 2>&1
done
for b in 0 4 3 2 1; do
  echo "== 8K band $b" >> gpurun_out/c4band.log
  if [ "$b" = 0 ]; then B=""; else B=$b; fi
  ILS_ROW_BAND=$B timeout 300 python tools/time_passes.py --h 4320 --w 7680 --reps 10 >> gpurun_out/c4band.log 2>&1
done
true
