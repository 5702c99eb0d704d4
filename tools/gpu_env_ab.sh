# A/B of environment settings on the C3 bench (interleaved twice): bash tools/gpu_env_ab.sh "" "ILS_COL2_SPEC=5" ...
: > gpurun_out/env_ab.log
for rep in 1 2; do
for e in "$@"; do
  echo "== [$e]" >> gpurun_out/env_ab.log
  env $e timeout 300 python bench.py --steps 30 --no-cpu --no-cufft --no-c4 --no-c5 --no-dropin --no-gray 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['col_pass']['frac'], d['roofline']['pass_ms_in_sequence'])" >> gpurun_out/env_ab.log 2>&1
done
done
cat gpurun_out/env_ab.log
