mkdir -p gpurun_out
: > gpurun_out/variants2.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for cfg in "default 2" "default 3" "minb4 2"; do
  set -- $cfg
  echo "== $1 streams $2" >> gpurun_out/variants2.log
  if [ "$1" = default ]; then L=""; else L=variants/$1.so; fi
  ILS_LIB=$L timeout 300 python tools/time_passes.py >> gpurun_out/variants2.log 2>&1
  ILS_LIB=$L timeout 300 python bench.py --steps 50 --streams $2 --no-cpu --no-cufft 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['pass_ms_in_sequence'])" >> gpurun_out/variants2.log 2>&1
done
true
