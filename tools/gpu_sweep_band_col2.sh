# sweep: row band x two-stage column kernel variant (ILS_ROW_BAND, ILS_COL2_SPEC), short bench each
mkdir -p gpurun_out
: > gpurun_out/sweep.log
for band in 6 5 7; do
  for spec in 5 0 1 2 4; do
    echo "== band=$band col2=$spec" >> gpurun_out/sweep.log
    ILS_ROW_BAND=$band ILS_COL2_SPEC=$spec timeout 300 python bench.py --steps 30 --no-cpu --no-cufft --no-c4 --no-c5 --no-dropin --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['pass_ms_in_sequence'])" >> gpurun_out/sweep.log 2>&1
  done
done
true
