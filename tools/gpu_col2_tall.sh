# two-stage column variants at 2160 / 4320 rows (pass timings), plus the bench's gray legs
mkdir -p gpurun_out
: > gpurun_out/col2_tall.log
for spec in 9 14 7 8; do
  ILS_COL2_SPEC=$spec timeout 300 python tools/time_passes.py --h 2160 --w 3840 >> gpurun_out/col2_tall.log 2>&1
done
for spec in 10 11 12; do
  ILS_COL2_SPEC=$spec timeout 300 python tools/time_passes.py --h 4320 --w 7680 --reps 10 >> gpurun_out/col2_tall.log 2>&1
done
timeout 600 python bench.py --steps 20 --no-cpu --no-cufft --no-c4 --no-c5 --no-dropin --no-e2e > gpurun_out/bench_gray.log 2>&1
true
