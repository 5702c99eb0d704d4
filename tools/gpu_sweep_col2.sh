mkdir -p gpurun_out
: > gpurun_out/sweep.log
for s in 5 11 12; do
  echo "spec $s" >> gpurun_out/sweep.log
  ILS_COL2_SPEC=$s timeout 300 python tools/time_passes.py >> gpurun_out/sweep.log 2>&1
  ILS_COL2_SPEC=$s timeout 300 python bench.py --steps 50 --no-cpu --no-cufft --no-e2e 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['pass_ms_in_sequence'])" >> gpurun_out/sweep.log 2>&1
done
ILS_COL2_SPEC=0 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "slab or c3 or launch_pass" >> gpurun_out/sweep.log 2>&1
true
