# time the bench and passes for each variants/*.so against the default build
mkdir -p gpurun_out
: > gpurun_out/variants.log
for lib in default variants/*.so; do
  echo "== $lib" >> gpurun_out/variants.log
  if [ "$lib" = default ]; then L=""; else L="$lib"; fi
  ILS_LIB=$L timeout 300 python tools/time_passes.py >> gpurun_out/variants.log 2>&1
  ILS_LIB=$L timeout 300 python bench.py --steps 50 --no-cpu --no-cufft --no-c4 --no-c5 --no-dropin 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['pass_ms_in_sequence'])" >> gpurun_out/variants.log 2>&1
done
if [ -n "$NCU_VARIANTS" ]; then
  for lib in default variants/*.so; do
    if [ "$lib" = default ]; then L=""; n=default; else L="$lib"; n=$(basename $lib .so); fi
    ILS_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --cache-control none --clock-control none -k regex:'k_row|k_col' -c 9 --csv --log-file gpurun_out/ncu_$n.csv python tools/time_u8.py --frames 1 > /dev/null 2>&1
  done
fi
true
