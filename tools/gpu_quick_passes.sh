# pass timings at 1080p / 4K / 8K and bench step shapes (frames per ils_smooth call)
mkdir -p gpurun_out
: > gpurun_out/passes.log
timeout 300 python tools/time_passes.py >> gpurun_out/passes.log 2>&1
timeout 300 python tools/time_passes.py --h 2160 --w 3840 >> gpurun_out/passes.log 2>&1
timeout 300 python tools/time_passes.py --h 4320 --w 7680 --reps 10 >> gpurun_out/passes.log 2>&1
: > gpurun_out/shapes.log
for args in "--group 1" "--group 2" "--group 2 --streams 1" "--group 4 --streams 1"; do
  echo "== $args" >> gpurun_out/shapes.log
  timeout 300 python bench.py --steps 30 --no-cpu --no-cufft --no-c4 --no-c5 --no-dropin $args 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['pass_ms_in_sequence'])" >> gpurun_out/shapes.log 2>&1
done
true
