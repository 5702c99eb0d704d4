mkdir -p gpurun_out
: > gpurun_out/lanes.log
for s in 1 2 3 4; do
  echo "streams $s" >> gpurun_out/lanes.log
  timeout 300 python bench.py --steps 50 --streams $s --no-cpu --no-cufft --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['clocks'])" >> gpurun_out/lanes.log 2>&1
done
echo "streams 2 frames 32" >> gpurun_out/lanes.log
timeout 300 python bench.py --steps 50 --streams 2 --frames 32 --no-cpu --no-cufft --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'])" >> gpurun_out/lanes.log 2>&1
true
