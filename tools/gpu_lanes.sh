mkdir -p gpurun_out
: > gpurun_out/lanes.log
for cfg in "--streams 2 --group 1" "--streams 1 --group 2" "--streams 2 --group 2" "--streams 1 --group 4"; do
  echo "$cfg" >> gpurun_out/lanes.log
  timeout 300 python bench.py --steps 50 $cfg --no-cpu --no-cufft --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'])" >> gpurun_out/lanes.log 2>&1
done
true
