: > gpurun_out/fin8k.log
for e in "ILS_X=0" "ILS_FIN_BAND=1" "ILS_FIN_BAND=2" "ILS_FIN_BAND=3" "ILS_FIN_BAND=4"; do
  echo "== [$e]" >> gpurun_out/fin8k.log
  env $e timeout 300 python tools/time_passes.py --h 4320 --w 7680 --reps 10 | grep -o '"row_fin.*' >> gpurun_out/fin8k.log 2>&1
  env $e timeout 300 python bench.py --steps 5 --no-cpu --no-cufft --no-e2e --no-c4 --no-dropin --no-gray 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5', d['c5']['value'])" >> gpurun_out/fin8k.log 2>&1
done
cat gpurun_out/fin8k.log
