mkdir -p gpurun_out
: > gpurun_out/c5pass.log
timeout 300 python tools/time_passes.py --h 4320 --w 7680 --reps 20 >> gpurun_out/c5pass.log 2>&1
ILS_NO_PDL=1 timeout 300 python tools/time_passes.py --h 4320 --w 7680 --reps 20 >> gpurun_out/c5pass.log 2>&1
for i in 1 2 3; do timeout 300 python tools/bench_c5.py --steps 20 >> gpurun_out/c5pass.log 2>&1; done
ILS_NO_PDL=1 timeout 300 python tools/bench_c5.py --steps 20 >> gpurun_out/c5pass.log 2>&1
true
