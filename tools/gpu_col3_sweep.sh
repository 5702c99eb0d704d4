# column-solve kernel choice: k_col3 specs vs k_col2 (ILS_COL3_SPEC=-1), passes + short bench each
mkdir -p gpurun_out
: > gpurun_out/col3_sweep.log
for spec in -2 -1 7 8 0 2; do
  echo "== ILS_COL3_SPEC=$spec" >> gpurun_out/col3_sweep.log
  ILS_COL3_SPEC=$spec timeout 300 python tools/time_passes.py >> gpurun_out/col3_sweep.log 2>&1
  ILS_COL3_SPEC=$spec timeout 300 python bench.py --steps 50 --no-cpu --no-cufft --no-c4 --no-c5 --no-dropin 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['pass_ms_in_sequence'], d['parity'])" >> gpurun_out/col3_sweep.log 2>&1
done
true
