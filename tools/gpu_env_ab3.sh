# env A/B (interleaved twice): per-pass times at 1080p / 4K / 8K and the bench with C4 + C5
# bash tools/gpu_env_ab3.sh "ILS_X=0" "ILS_ROW_PF_AHEAD=0"
: > gpurun_out/env_ab3.log
for rep in 1 2; do
for e in "$@"; do
  echo "== [$e]" >> gpurun_out/env_ab3.log
  env $e timeout 300 python tools/time_passes.py >> gpurun_out/env_ab3.log 2>&1
  env $e timeout 300 python tools/time_passes.py --h 2160 --w 3840 >> gpurun_out/env_ab3.log 2>&1
  env $e timeout 300 python tools/time_passes.py --h 4320 --w 7680 --reps 10 >> gpurun_out/env_ab3.log 2>&1
  env $e timeout 600 python bench.py --steps 20 --no-cpu --no-cufft --no-dropin --no-gray 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['pass_ms_in_sequence'], 'c4', d['c4']['value'], 'c5', d['c5']['value'])" >> gpurun_out/env_ab3.log 2>&1
done
done
grep -o "^== .*\|\"row_f0\".*\|bench.*" gpurun_out/env_ab3.log
