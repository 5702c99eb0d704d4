# ncu: rolling row pass vs k_row at 3840x2160 (IT pass), one launch each
mkdir -p gpurun_out
for roll in 0 1; do
  ILS_NO_ROLL=$((1-roll)) timeout 600 ncu --set full --import-source on --cache-control none --clock-control none -k regex:'k_row' --launch-skip 7 --launch-count 1 -o gpurun_out/roll_$roll python tools/time_passes.py --h 2160 --w 3840 --reps 1 > gpurun_out/ncu_roll_$roll.log 2>&1
done
true
