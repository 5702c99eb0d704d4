mkdir -p gpurun_out
: > gpurun_out/ingest.log
timeout 900 python -m pytest tests -m gpu -x -q >> gpurun_out/ingest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ingest.log
python - >> gpurun_out/ingest.log 2>&1 <<'PY'
import os, numpy as np, torch, paper_2003_07504_b200 as ils
rng = np.random.default_rng(9)
p = ils.SmoothParams(ils.Charbonnier(0.8, 1e-4), 1.0)
f8 = torch.from_numpy(rng.integers(0, 256, (2, 1080, 1920, 3), dtype=np.uint8)).cuda()
a = ils.smooth_frames_u8(f8, p)
planes = (f8.permute(0, 3, 1, 2).reshape(6, 1080, 1920).to(torch.float64) / 255.0).to(torch.float32)
u = ils.smooth_batch(planes, p)
q = torch.floor(torch.clamp(u, 0, 1) * 255 + 0.5).to(torch.uint8).reshape(2, 3, 1080, 1920).permute(0, 2, 3, 1)
print("fused ingest == planar path:", bool(torch.equal(a, q)), int((a.int() - q.int()).abs().max()))
PY
for v in 0 1 0 1; do
  echo "NO_FUSED=$v" >> gpurun_out/ingest.log
  ILS_NO_FUSED_INGEST=$v timeout 600 python bench.py --no-cpu --no-cufft 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'])" >> gpurun_out/ingest.log 2>&1
done
true
