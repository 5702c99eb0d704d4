mkdir -p gpurun_out
: > gpurun_out/hostgraph.log
timeout 600 python -m pytest tests -m gpu -x -q -k "u8 or host or app or e2e" >> gpurun_out/hostgraph.log 2>&1
for v in 1 0 1 0; do
  echo "HOST_GRAPHS=$v" >> gpurun_out/hostgraph.log
  ILS_HOST_GRAPHS=$v timeout 600 python bench.py --no-cpu --no-cufft 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e_f32_planes']['value'])" >> gpurun_out/hostgraph.log 2>&1
done
ILS_HOST_GRAPHS=1 timeout 300 python tools/e2e_probe.py 2>&1 | grep host >> gpurun_out/hostgraph.log
true
