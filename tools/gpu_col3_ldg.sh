mkdir -p gpurun_out
: > gpurun_out/col3_ldg.log
for lib in "" variants/c3ldg.so; do
  for spec in -1 7 0; do
    echo "== lib=$lib spec=$spec" >> gpurun_out/col3_ldg.log
    ILS_LIB=$lib ILS_COL3_SPEC=$spec timeout 300 python tools/time_passes.py >> gpurun_out/col3_ldg.log 2>&1
  done
  for spec in -1 9 4; do
    ILS_LIB=$lib ILS_COL3_SPEC=$spec timeout 300 python tools/time_passes.py --h 2160 --w 3840 >> gpurun_out/col3_ldg.log 2>&1
  done
  ILS_LIB=$lib ILS_COL3_SPEC=7 timeout 300 python bench.py --steps 50 --no-cpu --no-cufft --no-c4 --no-c5 --no-dropin 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['pass_ms_in_sequence'])" >> gpurun_out/col3_ldg.log 2>&1
done
true
