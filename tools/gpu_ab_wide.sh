mkdir -p gpurun_out
: > gpurun_out/ab4k.log
for lib in "" variants/rollminb1.so; do
  ILS_LIB=$lib timeout 300 python tools/time_passes.py --h 2160 --w 3840 >> gpurun_out/ab4k.log 2>&1
  ILS_LIB=$lib timeout 300 python tools/time_passes.py --h 4320 --w 7680 --reps 10 >> gpurun_out/ab4k.log 2>&1
done
timeout 300 python tools/time_passes.py >> gpurun_out/ab4k.log 2>&1
true
