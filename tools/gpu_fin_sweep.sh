: > gpurun_out/fin.log
for e in "ILS_X=0" "ILS_FIN_BAND=7" "ILS_FIN_BAND=5" "ILS_FIN_BAND=4" "ILS_FIN_BAND=3"; do
  echo "== [$e]" >> gpurun_out/fin.log
  env $e timeout 300 python tools/time_passes.py --h 2160 --w 3840 | grep -o '"row_band.*' >> gpurun_out/fin.log 2>&1
  for l in 1 2; do
  env $e ILS_C4_LANES=$l timeout 300 python bench.py --steps 5 --no-cpu --no-cufft --no-e2e --no-c5 --no-dropin --no-gray 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4 lanes', d['c4']['lanes'], d['c4']['value'])" >> gpurun_out/fin.log 2>&1
  done
done
cat gpurun_out/fin.log
