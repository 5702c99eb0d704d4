mkdir -p gpurun_out
: > gpurun_out/cl.log
for cfg in "6 0" "6 1" "7 0"; do
  set -- $cfg
  echo "== band $1 nocluster $2" >> gpurun_out/cl.log
  ILS_ROW_BAND=$1 ILS_NO_CLUSTER=$2 timeout 300 python tools/time_passes.py >> gpurun_out/cl.log 2>&1
  ILS_ROW_BAND=$1 ILS_NO_CLUSTER=$2 timeout 300 python bench.py --steps 50 --no-cpu --no-cufft 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['pass_ms_in_sequence'])" >> gpurun_out/cl.log 2>&1
done
ILS_ROW_BAND=6 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c3 or determinism or launch_pass" >> gpurun_out/cl.log 2>&1
true
