# time the bench and passes for each variants/*.so against the default build
mkdir -p gpurun_out
: > gpurun_out/variants.log
for lib in default variants/*.so; do
  echo "== $lib" >> gpurun_out/variants.log
  if [ "$lib" = default ]; then L=""; else L="$lib"; fi
  ILS_LIB=$L timeout 300 python tools/time_passes.py >> gpurun_out/variants.log 2>&1
  ILS_LIB=$L timeout 300 python bench.py --steps 50 --no-cpu --no-cufft 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['pass_ms_in_sequence'])" >> gpurun_out/variants.log 2>&1
done
true
