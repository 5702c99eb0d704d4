: > gpurun_out/frames.log
for rep in 1 2; do
for fr in 32 64 128; do
  echo "== frames $fr" >> gpurun_out/frames.log
  timeout 300 python bench.py --steps 30 --frames $fr --no-cpu --no-cufft --no-c4 --no-c5 --no-dropin --no-gray 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e']['ms_per_step'])" >> gpurun_out/frames.log 2>&1
done
done
cat gpurun_out/frames.log
