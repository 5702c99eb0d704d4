# 320-thread row CTAs (10 line groups) for the 1920-wide plan, 2 CTAs/SM, band 8 (10 lines = 10 warps)
: > gpurun_out/t320.log
for rep in 1 2; do
echo "== default" >> gpurun_out/t320.log
timeout 300 python bench.py --steps 30 --no-cpu --no-cufft --no-c4 --no-c5 --no-dropin --no-e2e --no-gray 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['pass_ms_in_sequence'])" >> gpurun_out/t320.log 2>&1
for band in 8 18; do
  echo "== t320 band=$band" >> gpurun_out/t320.log
  ILS_LIB=variants/t320.so ILS_ROW_BAND=$band timeout 300 python tools/time_passes.py >> gpurun_out/t320.log 2>&1
  ILS_LIB=variants/t320.so ILS_ROW_BAND=$band timeout 300 python bench.py --steps 30 --no-cpu --no-cufft --no-c4 --no-c5 --no-dropin --no-e2e --no-gray 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['pass_ms_in_sequence'], d['parity']['max_abs'])" >> gpurun_out/t320.log 2>&1
done
done
cat gpurun_out/t320.log
