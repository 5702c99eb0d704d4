# A/B: variants/*.so against the in-tree library (passes alone + short bench), interleaved twice
mkdir -p gpurun_out
: > gpurun_out/ab.log
for rep in 1 2; do
for lib in default variants/*.so; do
  echo "== $lib" >> gpurun_out/ab.log
  if [ "$lib" = default ]; then L=""; else L="$lib"; fi
  ILS_LIB=$L timeout 300 python tools/time_passes.py >> gpurun_out/ab.log 2>&1
  ILS_LIB=$L timeout 300 python bench.py --steps 30 --no-cpu --no-cufft --no-c4 --no-c5 --no-dropin 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['pass_ms_in_sequence'])" >> gpurun_out/ab.log 2>&1
done
done
true
