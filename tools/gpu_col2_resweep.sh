# col2 strip shapes per column height after the bulk-copied tables (per-pass times alone)
: > gpurun_out/col2_resweep.log
for id in 0 5 1 2 3 4 6; do echo "1080 spec $id" >> gpurun_out/col2_resweep.log; ILS_COL2_SPEC=$id timeout 120 python tools/time_passes.py >> gpurun_out/col2_resweep.log 2>&1; done
for id in 8 9 7 14; do echo "2160 spec $id" >> gpurun_out/col2_resweep.log; ILS_COL2_SPEC=$id timeout 120 python tools/time_passes.py --h 2160 --w 3840 >> gpurun_out/col2_resweep.log 2>&1; done
for id in 10 11 12; do echo "4320 spec $id" >> gpurun_out/col2_resweep.log; ILS_COL2_SPEC=$id timeout 200 python tools/time_passes.py --h 4320 --w 7680 --reps 10 >> gpurun_out/col2_resweep.log 2>&1; done
true
