mkdir -p gpurun_out
: > gpurun_out/pdl_ab.log
for i in 1 2; do
  for v in 0 1; do
    echo "NO_PDL=$v" >> gpurun_out/pdl_ab.log
    ILS_NO_PDL=$v timeout 600 python bench.py --no-cpu --no-cufft 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e_f32_planes']['value'])" >> gpurun_out/pdl_ab.log 2>&1
    ILS_NO_PDL=$v timeout 300 python tools/e2e_probe.py 2>&1 | grep -E "2 lane|nbatches=16" >> gpurun_out/pdl_ab.log
  done
done
true
