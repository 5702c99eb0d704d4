: > gpurun_out/roll4k.log
python -c "
import sys; sys.path.insert(0,'.')
import paper_2003_07504_b200 as ils
from paper_2003_07504_b200 import _lib, _runtime as rt
p = rt.get_plan(3, 2160, 3840, ils.SmoothParams(ils.Charbonnier(0.8,1e-4),1.0).c_params(), _lib.ILS_F32, 0)
print('default roll rows', p.info['row_roll_rows'])" >> gpurun_out/roll4k.log 2>&1
for rep in 1 2; do
for e in "ILS_X=0" "ILS_ROLL_PF=1" "ILS_ROLL_ROWS=6" "ILS_ROLL_ROWS=8" "ILS_ROLL_ROWS=10" "ILS_ROLL_PF=1 ILS_ROLL_ROWS=8"; do
  echo "== [$e]" >> gpurun_out/roll4k.log
  env $e timeout 300 python tools/time_passes.py --h 2160 --w 3840 | grep -o '"row_f0.*' >> gpurun_out/roll4k.log 2>&1
  env $e timeout 300 python bench.py --steps 5 --no-cpu --no-cufft --no-e2e --no-c5 --no-dropin --no-gray 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4', d['c4']['value'])" >> gpurun_out/roll4k.log 2>&1
done
done
cat gpurun_out/roll4k.log
