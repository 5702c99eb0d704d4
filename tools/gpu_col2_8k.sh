: > gpurun_out/col2_8k.log
for id in 10 11 12 15; do echo "4320 spec $id" >> gpurun_out/col2_8k.log; ILS_COL2_SPEC=$id timeout 200 python tools/time_passes.py --h 4320 --w 7680 --reps 10 >> gpurun_out/col2_8k.log 2>&1; done
for id in 8 7 14; do echo "2160 spec $id" >> gpurun_out/col2_8k.log; ILS_COL2_SPEC=$id timeout 120 python tools/time_passes.py --h 2160 --w 3840 >> gpurun_out/col2_8k.log 2>&1; done
grep -A1 spec gpurun_out/col2_8k.log | grep -o "[0-9]* spec [0-9]*\|\"col\": [0-9.]*" | paste - -
