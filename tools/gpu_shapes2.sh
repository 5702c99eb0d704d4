# bench shape sweep: lanes / frames per step (C3), lanes for C4
: > gpurun_out/shapes2.log
for a in "--streams 2" "--streams 3" "--streams 4" "--streams 2 --frames 64" "--streams 3 --frames 48"; do
  echo "== $a" >> gpurun_out/shapes2.log
  timeout 300 python bench.py --steps 30 --no-cpu --no-cufft --no-c4 --no-c5 --no-dropin --no-gray $a 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'])" >> gpurun_out/shapes2.log 2>&1
done
for l in 1 2; do
  echo "== c4 lanes $l" >> gpurun_out/shapes2.log
  ILS_C4_LANES=$l timeout 300 python bench.py --steps 5 --no-cpu --no-cufft --no-e2e --no-c5 --no-dropin --no-gray 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['c4']['value'])" >> gpurun_out/shapes2.log 2>&1
done
cat gpurun_out/shapes2.log
