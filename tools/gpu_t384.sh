# 384-thread row CTAs for the 1920-wide plan (2 CTAs/SM) over band sizes vs the default 256-thread band 6
mkdir -p gpurun_out
: > gpurun_out/t384.log
echo "== default" >> gpurun_out/t384.log
timeout 300 python bench.py --steps 30 --no-cpu --no-cufft --no-c4 --no-c5 --no-dropin --no-e2e --no-gray 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['pass_ms_in_sequence'])" >> gpurun_out/t384.log 2>&1
for band in 10 12 8 9 11; do
  echo "== t384 band=$band" >> gpurun_out/t384.log
  ILS_LIB=variants/t384.so ILS_ROW_BAND=$band timeout 300 python tools/time_passes.py >> gpurun_out/t384.log 2>&1
  ILS_LIB=variants/t384.so ILS_ROW_BAND=$band timeout 300 python bench.py --steps 30 --no-cpu --no-cufft --no-c4 --no-c5 --no-dropin --no-e2e --no-gray 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['pass_ms_in_sequence'], d['parity']['max_abs'])" >> gpurun_out/t384.log 2>&1
done
true
