"""Benchmark: 1080p colour ILS frames/s (N=4) on B200, plus HBM roofline fraction.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Workload (BASELINE.json configs[2], the metric's config): 1920x1080 RGB
frames, Charbonnier p=0.8, eps=1e-4, lambda=1, 4 iterations, c = c0.  A
"step" smooths a batch of F frames per GPU (synthetic uniform [0,1) planes,
rng.random as in the reference bench cli.py:270-273, generated on device).
F frames x 24.9 MB > L2, so each step's inputs stream from HBM; within a
frame group the working set (f + two half spectra, ~75 MB) stays in L2 across
the iterations, by design.  Frames shard across ranks with no communication
(scaling "weak").

value     device throughput: frames/s over all ranks, inputs resident in HBM,
          one CUDA-graph replay per step, CUDA events, max over ranks.
e2e       the same through the C ABI with HOST buffers (ils_smooth_host_u8):
          pinned host 8-bit RGB frames (the reference's PNG/PPM pixel format)
          -> device copies, kernels (v/255 deinterleave ahead of the first
          pass, the quantising store fused into the last), device -> host
          copies and the status readback inside the timed region, pipelined
          over frames.  e2e_f32_planes: the same with fp32 planes.
roofline  the dominant kernel (fused row pass, iterations >= 1), CUDA events
          around each of its launches inside the real per-frame pass
          sequence: algorithmic bytes / time vs the measured HBM copy
          bandwidth in MEASURED_PEAKS.json; `traffic` = ncu DRAM bytes per
          launch (profiles/traffic.json).  `issue`: the bound that binds --
          ncu warp instructions per launch / time vs 4 per SM per cycle.
cpu_baseline  the oracle port (numpy/scipy, the reference's own algorithm)
          on the host cores, one frame.
cufft     the same loop written with torch.fft.rfft2/irfft2 (cuFFT) and
          torch elementwise ops in fp32, one CUDA graph per step,
          timed in the same run; its output is checked against ours.
--impl reference  times that CPU path alone, as the driver's reference arm.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

H, W, CH, ITERS = 1080, 1920, 3, 4
P_EXP, EPS, LAM = 0.8, 1e-4, 1.0
METRIC = "1080p colour ILS frames/s (4 iters) on 1/2/4/8 B200; HBM roofline fraction"


def bytes_per_frame(iters=ITERS, h=H, w=W, ch=CH):
    """Algorithmic HBM bytes per frame: (20 N + 4) H W per plane (fp32)."""
    wc = w // 2 + 1
    spec = h * wc * 8
    plane = h * w * 4
    per_plane = (plane + spec) + iters * 2 * spec + (iters - 1) * (2 * spec + plane) + (spec + plane)
    return ch * per_plane


def measured_traffic(kernel, key="bytes"):
    """Per-launch DRAM bytes (or warp instructions) of `kernel` from the committed ncu capture, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return float(json.load(fh)[kernel][key])
    except Exception:
        return None


def issue_roofline(kernel, ms, sms, mhz):
    """The bound that actually binds: warp instructions per launch (ncu, committed) / event
    time vs the issue peak (4 schedulers x 1 warp-instruction/cycle per SM at the sampled clock)."""
    inst = measured_traffic(kernel, "warp_instructions")
    if inst is None or not mhz:
        return None
    achieved = inst / (ms / 1e3)
    peak = sms * 4 * mhz * 1e6
    return {"achieved": round(achieved / 1e9, 1), "peak": round(peak / 1e9, 1), "unit": "G warp-inst/s",
            "frac": round(achieved / peak, 4), "warp_instructions_per_launch": inst}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 50 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._p = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "50"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.15)  # let the first sample land before the timed region starts
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        time.sleep(0.06)
        self._p.terminate()
        try:
            out, _ = self._p.communicate(timeout=5)
        except Exception:
            self._p.kill()
            out, _ = self._p.communicate()
        for line in out.splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = sorted(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        smax = max((float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.strip().lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(self.rows)}


def cufft_loop(f, lam, iters, p, eps, c):
    """ILS with cuFFT + torch elementwise (comparison leg only, fp32, half spectra)."""
    import math

    import torch

    h, w = f.shape[-2:]
    wx = 2 - 2 * torch.cos(2 * math.pi * torch.arange(w // 2 + 1, device=f.device, dtype=torch.float64) / w)
    wy = 2 - 2 * torch.cos(2 * math.pi * torch.arange(h, device=f.device, dtype=torch.float64) / h)
    denom = (1 + c * lam / 2 * (wy[:, None] + wx[None, :])).float()
    ff = torch.fft.rfft2(f)

    def aux(x):
        return c * x - p * x * torch.pow(x * x + eps, p / 2 - 1)

    u = f
    for _ in range(iters):
        mx = aux(torch.roll(u, -1, -1) - u)
        my = aux(torch.roll(u, -1, -2) - u)
        a = torch.roll(mx, 1, -1) - mx + torch.roll(my, 1, -2) - my
        u = torch.fft.irfft2((ff + lam / 2 * torch.fft.rfft2(a)) / denom, s=(h, w))
    return u


def cpu_port_frame_seconds(frames=1, seed=20240607, warm=True):
    """Oracle port (the reference algorithm, numpy + scipy.fft) on one 1080p RGB frame."""
    from oracle import ils_oracle as O

    workers = os.cpu_count() or 1
    planes = O.bench_planes(H, W, CH, seed=seed)
    pen = O.Charbonnier(P_EXP, EPS)
    if warm:
        O.smooth_color(planes[:1], pen, LAM, ITERS, workers=workers)  # warm-up (plans, pages)
    t0 = time.perf_counter()
    for _ in range(frames):
        O.smooth_color(planes, pen, LAM, ITERS, workers=workers)
    return (time.perf_counter() - t0) / frames, workers


def run_reference(args, rank):
    """--impl reference: the reference's algorithm on host cores (oracle port)."""
    if rank != 0:
        return
    sec, workers = cpu_port_frame_seconds(frames=1)  # warm-up + one sample
    samples = []
    # each step is one 1080p RGB frame (~1 s on 16 cores): cap the sample so
    # the reference arm finishes within a few minutes at any --steps
    for _ in range(max(1, min(args.steps, 30))):
        s, _ = cpu_port_frame_seconds(frames=1, warm=False)
        samples.append(s)
    mean = sum(samples) / len(samples)
    fps = 1.0 / mean
    line = {
        "impl": "reference", "metric": METRIC, "value": round(fps, 4), "unit": "frames/s",
        "n_gpus": args.gpus, "steps": len(samples), "warmup": 1, "ms_per_step": round(mean * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C3: 1920x1080 RGB ILS, Charbonnier p=0.8 eps=1e-4 lambda=1, 4 iters",
                   "frames_per_step": 1, "impl": "oracle port of ilsmooth.smooth_color (numpy/scipy.fft)"},
        "cpu_baseline": {"value": round(fps, 4), "unit": "frames/s", "cores": workers, "kind": "port",
                         "sample": "1 frame (3 planes 1920x1080) per step; channels on a 3-thread pool, scipy.fft workers=cpu_count (smoother.py:208-210)"},
        "e2e": {"value": round(fps, 4), "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--frames", type=int, default=16, help="frames per step per GPU")
    ap.add_argument("--group", type=int, default=1, help="frames per ils_smooth call (L2-resident group)")
    ap.add_argument("--streams", type=int, default=2, help="concurrent frame-group lanes (graph branches)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cufft", action="store_true", help="skip the cuFFT + torch comparison leg")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_2003_07504_b200 as ils
    from paper_2003_07504_b200 import _lib, _runtime as rt

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    F = args.frames
    G = max(1, min(args.group, F))
    assert F % G == 0, "--frames must be a multiple of --group"
    params = ils.SmoothParams(ils.Charbonnier(P_EXP, EPS), LAM, iters=ITERS)
    cp = params.c_params()
    gen = torch.Generator(device=dev)
    gen.manual_seed(20240607 + rank)
    f = torch.rand((F * CH, H, W), generator=gen, device=dev, dtype=torch.float32)
    u = torch.empty_like(f)
    plan = rt.get_plan(G * CH, H, W, cp, _lib.ILS_F32, local)
    L = _lib.lib()
    S = max(1, args.streams)
    wss = [torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=dev) for _ in range(S)]
    stats = [torch.empty(1, dtype=torch.int32, device=dev) for _ in range(S)]
    ws, status = wss[0], stats[0]
    stream = torch.cuda.Stream(device=dev)
    lanes = [stream] + [torch.cuda.Stream(device=dev) for _ in range(S - 1)]
    ps = H * W

    def step_launches(s):
        # frame groups round-robin over S lanes forked from / joined to `s`
        for ln in lanes[1:]:
            ln.wait_stream(s)
        for gi, g0 in enumerate(range(0, F, G)):
            k = gi % S
            off = g0 * CH * ps * 4
            _lib.check(L.ils_smooth(plan.ptr, C.c_void_p(f.data_ptr() + off), C.c_void_p(u.data_ptr() + off), ps,
                                    C.c_void_p(wss[k].data_ptr()), C.c_void_p((s if k == 0 else lanes[k]).cuda_stream),
                                    C.c_void_p(stats[k].data_ptr()), None), "ils_smooth")
        for ln in lanes[1:]:
            s.wait_stream(ln)

    # ---- device throughput: one CUDA graph per step
    with torch.cuda.stream(stream):
        step_launches(stream)  # warm the plans / attributes outside capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        step_launches(stream)
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    for st_ in stats:
        rt.raise_status(int(st_.item()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(args.steps):
                graph.replay()
            e1.record(stream)
        barrier()
    ms_step = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    for st_ in stats:
        rt.raise_status(int(st_.item()))
    value = world * F / (ms_step / 1e3)
    launches = args.steps * (F // G) * plan.info["launches_per_call"]

    # ---- dominant kernel alone (fused row pass, iteration >= 1) and the column pass
    def time_pass(pass_id, reps=20):
        with torch.cuda.stream(stream):
            for _ in range(3):
                L.ils_launch_pass(plan.ptr, pass_id, C.c_void_p(f.data_ptr()), C.c_void_p(u.data_ptr()), ps,
                                  C.c_void_p(ws.data_ptr()), C.c_void_p(stream.cuda_stream),
                                  C.c_void_p(status.data_ptr()))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                _lib.check(L.ils_launch_pass(plan.ptr, pass_id, C.c_void_p(f.data_ptr()), C.c_void_p(u.data_ptr()),
                                             ps, C.c_void_p(ws.data_ptr()), C.c_void_p(stream.cuda_stream),
                                             C.c_void_p(status.data_ptr())), "ils_launch_pass")
            b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    def time_in_sequence(frames=4):
        """Per-kernel CUDA-event durations inside the real pass sequence (warm L2).

        Replays the per-frame order F0, col, (IT, col) x (N-1), FIN through
        ils_launch_pass with an event pair around every launch.
        """
        order = [0, 1]
        for n in range(1, ITERS):  # current spectrum alternates A/B (pass | 4 = B current)
            cur = 0 if n % 2 else 4
            order += [2 | cur, 1 | (cur ^ 4)]
        order += [3 | (0 if ITERS % 2 else 4)]
        acc = {p: [] for p in (0, 1, 2, 3)}
        with torch.cuda.stream(stream):
            for rep in range(2):  # first pass warms plans and L2
                # hold the stream while the launches are queued, so no host
                # submission gap lands between an event pair
                torch.cuda._sleep(200_000_000)
                evs = []
                for fr in range(frames):
                    off = (fr % (F // G)) * G * CH * ps * 4
                    for p in order:
                        a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a_.record(stream)
                        _lib.check(L.ils_launch_pass(plan.ptr, p, C.c_void_p(f.data_ptr() + off),
                                                     C.c_void_p(u.data_ptr() + off), ps, C.c_void_p(ws.data_ptr()),
                                                     C.c_void_p(stream.cuda_stream), C.c_void_p(status.data_ptr())),
                                   "ils_launch_pass")
                        b_.record(stream)
                        evs.append((p, a_, b_))
                torch.cuda.synchronize()
                if rep == 1:
                    for p, a_, b_ in evs:
                        acc[p & 3].append(a_.elapsed_time(b_))
        return {p: sum(v) / len(v) for p, v in acc.items()}

    u_graph = u[:CH].clone()
    seq = time_in_sequence()
    # the per-pass replay is the real dataflow: it reproduces the graph's output bit for bit
    assert torch.equal(u[:CH], u_graph), "per-pass sequence differs from ils_smooth"
    ms_row, ms_col = seq[2], seq[1]
    ms_row_isolated, ms_col_isolated = time_pass(2), time_pass(1)
    wc = W // 2 + 1
    planes_g = G * CH
    row_bytes = planes_g * (2 * H * wc * 8 + H * W * 4)
    col_bytes = planes_g * (2 * H * wc * 8)
    peak, peak_kind = peaks()
    row_gbs = row_bytes / (ms_row / 1e3) / 1e9
    col_gbs = col_bytes / (ms_col / 1e3) / 1e9

    # ---- end to end through the C ABI with pinned host buffers
    def e2e_leg(u8):
        """ils_smooth_host(_u8): pinned host frames in, results out, copies in the timed region."""
        if u8:
            gen8 = torch.Generator(device=dev)
            gen8.manual_seed(20240607 + rank)
            fd8 = torch.randint(0, 256, (F, H, W, CH), generator=gen8, device=dev, dtype=torch.uint8)
            fh = torch.empty((F, H, W, CH), dtype=torch.uint8, pin_memory=True)
            fh.copy_(fd8.cpu())
        else:
            fh = torch.empty((F * CH, H, W), dtype=torch.float32, pin_memory=True)
            fh.copy_(f.cpu())
        uh = torch.empty_like(fh, pin_memory=True)
        io = C.c_size_t()
        _lib.check(L.ils_host_io_size(plan.ptr, C.byref(io)), "ils_host_io_size")
        iobuf = torch.empty(io.value, dtype=torch.uint8, device=dev)
        bad = C.c_int32()

        def host_call():
            if u8:
                _lib.check(L.ils_smooth_host_u8(plan.ptr, C.c_void_p(fh.data_ptr()), C.c_void_p(uh.data_ptr()), CH,
                                                F // G, C.c_void_p(ws.data_ptr()), C.c_void_p(iobuf.data_ptr()),
                                                C.c_void_p(stream.cuda_stream), C.byref(bad)), "ils_smooth_host_u8")
            else:
                _lib.check(L.ils_smooth_host(plan.ptr, C.c_void_p(fh.data_ptr()), C.c_void_p(uh.data_ptr()), ps,
                                             F // G, C.c_void_p(ws.data_ptr()), C.c_void_p(iobuf.data_ptr()),
                                             C.c_void_p(stream.cuda_stream), C.byref(bad)), "ils_smooth_host")

        for _ in range(max(1, args.warmup)):
            host_call()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2e_steps = max(1, args.steps // 2)
        a.record(stream)
        for _ in range(e2e_steps):
            host_call()
        b.record(stream)
        barrier()
        ms_e2e = max_over_ranks(a.elapsed_time(b) / e2e_steps)
        if u8:  # the fused 8-bit path equals the device path on the same frames
            got = ils.smooth_frames_u8(fd8[:G], params)
            assert torch.equal(uh[:G].to(dev), got), "e2e output differs from device path"
            nbytes = F * CH * H * W
            api = "ils_smooth_host_u8 (C ABI): pinned host 8-bit RGB frames in and out (the reference's PNG/PPM pixel path)"
        else:
            assert torch.equal(uh[:CH].to(dev), u[:CH]), "e2e output differs from device path"
            nbytes = F * CH * H * W * 4
            api = "ils_smooth_host (C ABI): pinned host fp32 planes in and out"
        return {"value": round(world * F / (ms_e2e / 1e3), 2), "unit": "frames/s",
                "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes + (F // G) * 4,
                "ms_per_step": round(ms_e2e, 3), "api": api}

    e2e = e2e_f32 = None
    if not args.no_e2e:
        e2e = e2e_leg(u8=True)
        e2e_f32 = e2e_leg(u8=False)

    # ---- comparison: the same loop on cuFFT + torch elementwise, same frames
    cufft = None
    if not args.no_cufft:
        cpar = params.curvature
        fg = f[: G * CH * 2]  # two groups per call, like the two lanes
        with torch.cuda.stream(stream):
            ref_u = cufft_loop(fg, LAM, ITERS, P_EXP, EPS, cpar)
            torch.cuda.synchronize()
            gref = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gref, stream=stream):
                out_ref = cufft_loop(fg, LAM, ITERS, P_EXP, EPS, cpar)
            for _ in range(3):
                gref.replay()
            reps = max(3, args.steps // 4)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                gref.replay()
            b.record(stream)
        torch.cuda.synchronize()
        ms_ref = max_over_ranks(a.elapsed_time(b) / reps)
        diff = float((out_ref - u[: fg.shape[0]]).abs().max())
        cufft = {"value": round(world * (fg.shape[0] // CH) / (ms_ref / 1e3), 2), "unit": "frames/s",
                 "impl": "torch.fft.rfft2/irfft2 (cuFFT) + torch elementwise, fp32, CUDA graph",
                 "max_abs_diff_vs_ours": diff}
        del ref_u

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sec, workers = cpu_port_frame_seconds(frames=1)
        cpu = {"value": round(1.0 / sec, 4), "unit": "frames/s", "cores": workers, "kind": "port",
               "sample": "1 frame (3 planes 1920x1080), oracle port of smooth_color: channels on a 3-thread pool, scipy.fft workers=cpu_count (smoother.py:208-210)"}

    if rank == 0:
        bpf = bytes_per_frame()
        clk_sum = clk.summary()
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": "C3: 1920x1080 RGB ILS, Charbonnier p=0.8 eps=1e-4 lambda=1, 4 iters",
                       "frames_per_step_per_gpu": F, "frames_per_launch_group": G, "streams": S,
                       "parallelism": f"frame-sharded x{world}", "l2": "inputs larger than L2 (F x 24.9 MB)",
                       "plan": {k: plan.info[k] for k in ("row_band", "row_group", "row_radix", "row_spec", "col2_spec",
                                                          "col2_n1", "col2_n2", "col2_cols")}},
            "e2e": e2e,
            "e2e_f32_planes": e2e_f32,
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": round(row_gbs, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(row_gbs / peak, 4), "traffic": measured_traffic("k_row_it"),
                         "traffic_source": "profiles/traffic.json (ncu --set full, warm L2)", "peak_kind": peak_kind,
                         "issue": issue_roofline("k_row_it", ms_row, sms, clk_sum["sm_mhz"]),
                         "kernel": "k_row fused row pass (iteration>=1)", "ms": round(ms_row, 4),
                         "timing": "CUDA events around each launch inside the per-frame pass sequence (warm L2)",
                         "ms_isolated_loop": round(ms_row_isolated, 4),
                         "pass_ms_in_sequence": {"row_f0": round(seq[0], 4), "col": round(seq[1], 4),
                                                 "row_it": round(seq[2], 4), "row_fin": round(seq[3], 4)},
                         "bytes_per_launch": row_bytes,
                         "col_pass": {"kernel": "k_col2" if plan.info.get("col2_spec", -1) >= 0 else "k_col",
                                      "achieved": round(col_gbs, 1), "frac": round(col_gbs / peak, 4),
                                      "traffic": measured_traffic("k_col2" if plan.info.get("col2_spec", -1) >= 0
                                                                  else "k_col"),
                                      "issue": issue_roofline("k_col2", ms_col, sms, clk_sum["sm_mhz"])
                                      if plan.info.get("col2_spec", -1) >= 0 else None,
                                      "ms": round(ms_col, 4), "ms_isolated_loop": round(ms_col_isolated, 4),
                                      "bytes_per_launch": col_bytes},
                         "whole_path": {"achieved": round(bpf * value / world / 1e9, 1),
                                        "frac": round(bpf * value / world / 1e9 / peak, 4),
                                        "bytes_per_frame": bpf}},
            "cpu_baseline": cpu,
            "cufft_comparison": cufft,
            "clocks": clk_sum,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
