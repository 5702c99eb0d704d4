mkdir -p gpurun_out
: > gpurun_out/c5pass.log
for i in 1 2; do
timeout 300 python tools/time_passes.py --h 4320 --w 7680 --reps 20 >> gpurun_out/c5pass.log 2>&1
ILS_NO_COL2=1 timeout 300 python tools/time_passes.py --h 4320 --w 7680 --reps 20 >> gpurun_out/c5pass.log 2>&1
timeout 300 python tools/time_passes.py --h 2160 --w 3840 --reps 20 >> gpurun_out/c5pass.log 2>&1
ILS_NO_COL2=1 timeout 300 python tools/time_passes.py --h 2160 --w 3840 --reps 20 >> gpurun_out/c5pass.log 2>&1
done
true
