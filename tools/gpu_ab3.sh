# A/B of variants/*.so against the in-tree library: per-pass times at 1080p, 4K and 8K,
# then the bench (C3 + C4 + C5 legs) for each
mkdir -p gpurun_out
: > gpurun_out/ab3.log
for rep in 1 2; do for lib in default variants/*.so; do
  if [ "$lib" = default ]; then L=""; else L="$lib"; fi
  echo "== $lib" >> gpurun_out/ab3.log
  ILS_LIB=$L timeout 300 python tools/time_passes.py >> gpurun_out/ab3.log 2>&1
  ILS_LIB=$L timeout 300 python tools/time_passes.py --h 2160 --w 3840 >> gpurun_out/ab3.log 2>&1
  ILS_LIB=$L timeout 300 python tools/time_passes.py --h 4320 --w 7680 --reps 10 >> gpurun_out/ab3.log 2>&1
  ILS_LIB=$L timeout 600 python bench.py --steps 20 --no-cpu --no-cufft --no-dropin --no-gray 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['pass_ms_in_sequence'], 'c4', d['c4']['value'], 'c5', d['c5']['value'])" >> gpurun_out/ab3.log 2>&1
done; done
true
