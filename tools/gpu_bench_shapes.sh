# bench step shapes: frames per step x lanes (device value and host-pipeline e2e)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rowroll.py -q -p no:cacheprovider > gpurun_out/pytest_roll.log 2>&1
: > gpurun_out/shapes.log
for args in "--frames 16 --streams 2" "--frames 32 --streams 2" "--frames 16 --streams 3" "--frames 32 --streams 3" "--frames 24 --streams 3" "--frames 32 --streams 4"; do
  echo "== $args" >> gpurun_out/shapes.log
  timeout 300 python bench.py --steps 30 --no-cpu --no-cufft --no-c4 --no-c5 --no-dropin $args 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e_f32_planes']['value'])" >> gpurun_out/shapes.log 2>&1
done
true
