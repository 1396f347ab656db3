#!/usr/bin/env python
"""Benchmark of the B200 coarse pose-search hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[1]): one 1024x768 uint8 image
pair at transition tilt (t1=4 @0deg vs t2=4*sqrt2 @90deg), the reference's
default viewpoint grid (a=sqrt2, n=5, b=72deg, delta_s=0.5 -> 43 views),
Lanczos-4 views, ORB 1000 keypoints/view, 8 levels x1.2, FAST 20, ratio 0.8.
One step = one coarse_search over the pair: target ORB + 43 x (anti-alias blur
-> Lanczos view -> uint8 -> ORB detect -> content filter -> describe ->
Hamming ratio count). Metric: views/s (whole job). Under torchrun every rank
runs its own pair (seed + rank): weak scaling, counts gathered over NCCL.

value: device time of the step with inputs resident in HBM (CUDA events on the
engine stream; L2 flushed between steps with a 256 MiB write, not timed).
e2e:   the public host API (xa_coarse_search) with pinned host buffers: H2D of
the pair, the step, D2H of the counts, wall clock per step.
Secondary (same line): BASELINE configs[3] Hamming 200k x 200k comparisons/s.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import pathlib
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "affine views/s (Lanczos warp+ORB) at 1/2/4/8 B200; Hamming comparisons/s"
WORKLOAD = ("config2: 1024x768 uint8 pair, transition tilt t1=4@0deg vs t2=4sqrt2@90deg; "
            "grid a=sqrt2 n=5 b=72deg delta_s=0.5 (43 views); Lanczos-4 views quantised to uint8; "
            "ORB 1000 kp/view, 8 levels x1.2, FAST 20 (auto-relax 7); BF Hamming k=2 ratio 0.8")
MAX_POINTS, RATIO = 1000, 0.8


def peaks():
    p = {}
    try:
        p = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    return p


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        rows = []
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) >= 9:
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][2]), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows)}


def stage_work(xa, grid, w, h, counters):
    """Algorithmic work per stage for one step: FLOPs or bytes."""
    lanczos_px = 0.0
    out_px = 0
    blur_flop = 0.0
    view_px = []
    for p in grid.entries:
        m = xa.simulation_from_params(p)
        det = abs(m[0, 0] * m[1, 1] - m[0, 1] * m[1, 0])
        lanczos_px += det * (w - 1) * (h - 1)
        import ctypes as C
        from paper_2503_03479_b200 import _lib
        W, H, tx, ty = C.c_int(), C.c_int(), C.c_double(), C.c_double()
        mm = np.ascontiguousarray(m.reshape(-1))
        _lib.lib().xa_warp_frame(mm.ctypes.data_as(C.c_void_p), w, h, C.byref(W), C.byref(H),
                                 C.byref(tx), C.byref(ty), None)
        out_px += W.value * H.value
        view_px.append(W.value * H.value)
        if p.tilt != 1.0:
            sigma = 0.8 * math.sqrt(p.tilt ** 2 - 1)
            taps = 2 * max(1, math.ceil(3 * sigma)) + 1
            blur_flop += w * h * taps * (2 if p.phi == 0.0 else 8)
    pyr_px = 0
    for px in [w * h] + view_px:
        pyr_px += px * 3.10
    ncand = int(counters[:, 0].sum())
    ndesc = counters[:, 4]
    cmps = float(ndesc[1:].sum()) * float(ndesc[0])
    return {
        "antialias": ("fp32", blur_flop),
        # 128 FLOP per output px (64 MAC) over the view frames the
        # launch writes (W x H each; ~62% of them lie inside the content)
        "warp": ("fp32", 128.0 * out_px),
        # levels 1.. written + float level 0 of each view read once (the views'
        # level 0 is written by the resampler), + the uint8 target read
        "pyramid": ("hbm", pyr_px * 4 + w * h),
        "fast_nms": ("hbm", pyr_px * 4),
        "measures": ("fp64", ncand * 49 * 6.0),  # Harris: 3 DMUL + 3 DADD per window position
        "describe": ("fp32", float(ndesc.sum()) * 2 * 13 * (49 * 37 + 37 * 37)),
        "match": ("popc", 8.0 * cmps),
    }, {"lanczos_px": lanczos_px, "view_px": out_px, "pyramid_px": pyr_px, "comparisons": cmps,
        "candidates": ncand, "candidates_max": int(counters[:, 0].max()),
        "candidates_per_image": [int(c) for c in counters[:, 0]]}


def peak_for(kind, sms, mhz, pk):
    if kind == "hbm":
        return pk.get("hbm_gbs", 6650.0), "GB/s", "measured copy bandwidth (MEASURED_PEAKS.json)"
    if kind == "fp32":
        return 2 * 128 * sms * mhz * 1e6 / 1e12, "TFLOP/s", f"nominal FP32 ({sms} SMs x 128 lanes x 2 x {mhz:.0f} MHz)"
    if kind == "fp64":
        return 2 * 64 * sms * mhz * 1e6 / 1e12, "TFLOP/s", f"nominal FP64 ({sms} SMs x 64 lanes x 2 x {mhz:.0f} MHz)"
    if kind == "popc":
        return 16 * sms * mhz * 1e6 / 1e12, "Tpopc/s", f"nominal POPC ({sms} SMs x 16/clk x {mhz:.0f} MHz)"
    raise ValueError(kind)


def cpu_baseline_run(grid_rows, a, b, threads, kind=None):
    """Bounded CPU sample of the same workload: the reference (oracle/_ref) or its
    restatement, Lanczos views, all threads; returns (views/s, info)."""
    from oracle.oracle import Oracle, available
    kind = kind or ("reference" if available("reference") else "port")
    O = Oracle(kind)
    sub = grid_rows[::4]
    t0 = time.perf_counter()
    O.coarse_search(a.astype(np.float32), b.astype(np.float32), sub, MAX_POINTS, RATIO, "lanczos",
                    threads=threads)
    dt = time.perf_counter() - t0
    return len(sub) / dt, {"kind": kind, "cores": threads,
                           "sample": f"config2 pair, {len(sub)} of 43 grid entries (every 4th) + target ORB, "
                                     f"Lanczos views, {threads} threads, {dt:.2f} s wall (~{dt * threads:.0f} core-s)"}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation on the host cores."""
    if rank != 0:
        return
    from paper_2503_03479_b200 import synth
    from oracle.oracle import available
    a, b = synth.config2(seed=2)
    from oracle.oracle import Oracle
    kind = "reference" if available("reference") else "port"
    O = Oracle(kind)
    grid_rows = O.build_grid()
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_baseline_run(grid_rows, a, b, threads, kind)
    vals = [cpu_baseline_run(grid_rows, a, b, threads, kind) for _ in range(args.steps)]
    v = float(np.median([x[0] for x in vals]))
    info = vals[-1][1]
    print(json.dumps({
        "metric": METRIC, "value": v, "unit": "views/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * len(grid_rows[::4]) / v,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": WORKLOAD, "sample": info["sample"]},
        "cpu_baseline": {"value": v, "unit": "views/s", "cores": threads, "kind": kind,
                         "sample": info["sample"]},
        "e2e": {"value": v, "unit": "views/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def hamming_secondary(xa, eng, torch, dev, stream, pk, sms, mhz, steps=3):
    from paper_2503_03479_b200 import synth
    q, t, _, _ = synth.config4(200_000)
    n = len(q)
    dq = torch.from_numpy(q.view(np.int64)).to(dev)
    dt = torch.from_numpy(t.view(np.int64)).to(dev)
    bi = torch.empty(n, dtype=torch.int32, device=dev)
    bd = torch.empty(n, dtype=torch.int16, device=dev)
    sd = torch.empty(n, dtype=torch.int16, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    run = lambda: eng.match_hamming_device(dq.data_ptr(), n, dt.data_ptr(), n, RATIO, bi.data_ptr(),
                                           bd.data_ptr(), sd.data_ptr(), cnt.data_ptr(), stream.cuda_stream)
    run()
    torch.cuda.synchronize(dev)
    tot = 0.0
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    ms = tot / steps
    cmp_s = float(n) * n / (ms / 1e3)
    peak, unit, src = peak_for("popc", sms, mhz, pk)
    ach = 8.0 * n * n / (ms / 1e3) / 1e12
    return {"config": "config4: 200000 x 200000 uniform 256-bit, 20% planted (0-40 flips), k=2, ratio 0.8",
            "value": cmp_s, "unit": "Hamming comparisons/s", "ms": ms, "matches": int(cnt.item()),
            "roofline": {"bound": "popc", "achieved": ach, "peak": peak, "unit": unit,
                         "frac": ach / peak, "peak_source": src}}


def l2_secondary(xa, eng, torch, dev, stream, pk, sms, mhz, steps=3, n=4096):
    """Fine-stage L2 ratio matcher (sift.cpp:388-418): n x n
    SIFT-like 128-float descriptors, 3 lane-ops per dimension (sub, mul, add:
    the reference's rounding forbids FMA)."""
    rng = np.random.default_rng(3)
    a = rng.gamma(0.6, 1.0, size=(n, 128)).astype(np.float32)
    a = 512.0 * a / np.linalg.norm(a, axis=1, keepdims=True)
    b = a[rng.permutation(n)] + rng.normal(0, 3.0, size=(n, 128)).astype(np.float32)
    da, db = torch.from_numpy(a.astype(np.float32)).to(dev), torch.from_numpy(b).to(dev)
    bi = torch.empty(n, dtype=torch.int32, device=dev)
    dd = torch.empty(n, dtype=torch.float32, device=dev)
    kp = torch.empty(n, dtype=torch.uint8, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    run = lambda: eng.match_ratio_device(da.data_ptr(), n, db.data_ptr(), n, RATIO, bi.data_ptr(),
                                         dd.data_ptr(), kp.data_ptr(), cnt.data_ptr(), stream.cuda_stream)
    run()
    torch.cuda.synchronize(dev)
    tot = 0.0
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    ms = tot / steps
    peak = 128 * sms * mhz * 1e6 / 1e12
    ach = 384.0 * n * n / (ms / 1e3) / 1e12
    return {"config": f"fine-stage L2 ratio matcher: {n} x {n} SIFT-like 128-float descriptors, ratio 0.8",
            "value": float(n) * n / (ms / 1e3), "unit": "L2 comparisons/s", "ms": ms,
            "matches": int(cnt.item()),
            "roofline": {"bound": "fp32 lane-ops", "achieved": ach, "peak": peak, "unit": "Tops/s",
                         "frac": ach / peak,
                         "peak_source": f"nominal FP32 lane-ops ({sms} SMs x 128 x {mhz:.0f} MHz; no FMA)"}}


def fine_secondary(xa, eng, a, b, with_cpu=True, steps=3):
    """Fine stage (pipeline.cpp:154-190 without RANSAC) on
    the config-2 pair: SIFT detect + describe on both images + L2 ratio match,
    through the host API (uploads and readbacks included), timed on the host;
    the reference's own sift.cpp path (oracle/_ref, one thread) beside it."""
    af, bf = a.astype(np.float32), b.astype(np.float32)

    def gpu():
        ka, da = xa.describe_gradient(af, xa.detect_dog_keypoints(af, 2000, engine=eng), engine=eng)
        kb, db = xa.describe_gradient(bf, xa.detect_dog_keypoints(bf, 2000, engine=eng), engine=eng)
        return len(ka), len(kb), len(xa.match_ratio(da, db, 0.8, engine=eng))
    gpu()
    t0 = time.perf_counter()
    for _ in range(steps):
        na, nb, nm = gpu()
    g_ms = 1e3 * (time.perf_counter() - t0) / steps
    out = {"config": "fine stage on the config-2 pair: SIFT detect (2000) + describe on both images, "
                     "L2 ratio 0.8; host API incl. transfers",
           "value": 1e3 / g_ms, "unit": "image pairs/s", "ms": g_ms,
           "keypoints": [na, nb], "matches": nm}
    if with_cpu:
        from oracle.oracle import Oracle, available
        if available("reference"):
            R = Oracle("reference")
            t0 = time.perf_counter()
            ka, da = R.describe_gradient(af, R.detect_dog(af, 2000))
            kb, db = R.describe_gradient(bf, R.detect_dog(bf, 2000))
            R.match_ratio(da, db, 0.8)
            c_ms = 1e3 * (time.perf_counter() - t0)
            out["cpu_reference"] = {"value": 1e3 / c_ms, "unit": "image pairs/s", "ms": c_ms, "cores": 1,
                                    "kind": "reference"}
    return out


def asift_secondary(xa, eng, a, b, with_cpu=True):
    """Dual-simulation ASIFT baseline (pipeline.cpp:298-343
    without RANSAC) on the config-2 pair through the host API: the full
    reference grid (43 entries, scale 1) on both images, SIFT (1000 kp) per
    view, 43 x 43 L2 ratio matchings, duplicate merge. The reference's own
    path (oracle/_ref, one thread) is timed on the n=2 grid (10 x 10 views),
    with the device timed on the same reduced grid beside it."""
    af, bf = a.astype(np.float32), b.astype(np.float32)
    full = xa.build_param_grid(xa.GridConfig())
    small = xa.build_param_grid(xa.GridConfig(n=2))

    def gpu(grid):
        t0 = time.perf_counter()
        m = xa.asift_correspondences(af, bf, grid, 1000, 0.75, engine=eng)
        return 1e3 * (time.perf_counter() - t0), len(m)
    gpu(small)
    g_ms, nm = gpu(full)
    s_ms, ns = gpu(small)
    out = {"config": "ASIFT baseline on the config-2 pair: 43 + 43 Lanczos views (scale 1), SIFT 1000 kp "
                     "per view, 43 x 43 L2 ratio 0.75 matchings, 2-px duplicate merge; host API incl. "
                     "transfers", "value": 1e3 / g_ms, "unit": "image pairs/s", "ms": g_ms,
           "correspondences": nm,
           "reduced_grid": {"views": len(small.entries), "ms": s_ms, "correspondences": ns}}
    if with_cpu:
        from oracle.oracle import Oracle, available
        if available("reference"):
            R = Oracle("reference")
            g = np.array([[p.psi, p.tilt, p.phi, p.scale, p.tx, p.ty] for p in small.entries])
            t0 = time.perf_counter()
            r = R.asift_correspondences(af, bf, g, 1000, 0.75)
            c_ms = 1e3 * (time.perf_counter() - t0)
            out["cpu_reference_reduced_grid"] = {"ms": c_ms, "cores": 1, "kind": "reference",
                                                 "correspondences": len(r), "views": len(g)}
    return out


def synth_secondary(xa, eng, a, with_cpu=True, steps=5):
    """The harness's projective Lanczos render (eval.cpp:101-141)
    of the config-2 reference image under a perspective homography, through the
    host API (upload + render + readback); the reference's eval.cpp on one host
    core beside it."""
    af = a.astype(np.float32)
    hm = np.array([[0.85, -0.3, 20.0], [0.25, 0.9, -10.0], [2e-4, -1.5e-4, 1.0]])
    img, _ = xa.synth_warp_case(af, hm, engine=eng)
    t0 = time.perf_counter()
    for _ in range(steps):
        img, _ = xa.synth_warp_case(af, hm, engine=eng)
    g_ms = 1e3 * (time.perf_counter() - t0) / steps
    out = {"config": f"synth_warp_case: config-2 reference image {af.shape[1]}x{af.shape[0]} under a "
                     f"perspective homography -> {img.shape[1]}x{img.shape[0]} float, Lanczos-4; "
                     "host API incl. transfers",
           "value": 1e3 / g_ms, "unit": "renders/s", "ms": g_ms,
           "output_mpx_per_s": img.size / (g_ms * 1e3)}
    if with_cpu:
        from oracle.oracle import Oracle, available
        if available("reference"):
            R = Oracle("reference")
            t0 = time.perf_counter()
            R.synth_warp_case(af, hm)
            c_ms = 1e3 * (time.perf_counter() - t0)
            out["cpu_reference"] = {"value": 1e3 / c_ms, "unit": "renders/s", "ms": c_ms, "cores": 1,
                                    "kind": "reference"}
    return out


def views_secondary(xa, eng, torch, dev, stream, pk, sms, mhz, steps=3):
    """BASELINE configs[2]: one 4096^2 uint8 texture -> anti-alias blur + Lanczos-4
    -> uint8 views over the reference grid with delta_s = 0 (43 views: the
    reference sampling rule cannot produce the config's "64")."""
    from paper_2503_03479_b200 import synth
    src = synth.config3()
    n0 = 4096
    grid = xa.build_param_grid(xa.GridConfig(delta_s=0.0))
    offs, ws, hs, total = eng.simulate_views_plan(n0, n0, grid, 1)
    d_src = torch.from_numpy(src).to(dev)
    d_out = torch.empty(total, dtype=torch.uint8, device=dev)
    run = lambda: eng.simulate_views_device(d_src.data_ptr(), n0, n0, grid, 1, d_out.data_ptr(),
                                            stream.cuda_stream)
    run()
    torch.cuda.synchronize(dev)
    tot = 0.0
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run()
        e1.record(stream)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    ms = tot / steps
    nv = len(grid.entries)
    out_px = float(np.sum(ws.astype(np.int64) * hs))
    # algorithmic FLOPs: Lanczos 128 per in-domain output px, blur 8 per bilinear tap
    lz, bl = 0.0, 0.0
    for p in grid.entries:
        m = xa.simulation_from_params(p)
        lz += 128.0 * abs(m[0, 0] * m[1, 1] - m[0, 1] * m[1, 0]) * (n0 - 1) ** 2
        if p.tilt != 1.0:
            taps = 2 * max(1, math.ceil(3 * 0.8 * math.sqrt(p.tilt ** 2 - 1))) + 1
            bl += n0 * n0 * taps * (2 if p.phi == 0.0 else 8)
    peak, unit, src_s = peak_for("fp32", sms, mhz, pk)
    ach = (lz + bl) / (ms / 1e3) / 1e12
    return {"config": "config3: 4096x4096 uint8 texture -> 43 views (grid n=5, delta_s=0), "
                      "directional anti-alias blur + Lanczos-4, uint8 output",
            "value": nv / (ms / 1e3), "unit": "views/s", "ms": ms,
            "output_mpx_per_s": out_px / (ms / 1e3) / 1e6,
            "roofline": {"bound": "fp32", "achieved": ach, "peak": peak, "unit": unit,
                         "frac": ach / peak, "peak_source": src_s}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--mode", default="lanczos", choices=["lanczos", "nearest"])
    ap.add_argument("--no-stage-events", action="store_true",
                    help="time the graph without per-stage event nodes (no stage_ms/roofline)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    from paper_2503_03479_b200 import dist as D
    rank, world, local = D.init_from_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import paper_2503_03479_b200 as xa
    from paper_2503_03479_b200 import synth
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    coll_dev = dev
    if world > 1:
        import torch.distributed as dist
        if dist.get_backend() == "gloo":  # XA_DIST_BACKEND=gloo: CPU collectives
            coll_dev = torch.device("cpu")
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    pk = peaks()
    mhz = pk.get("sm_max_mhz", 1965.0)

    a, b = synth.config2(seed=2 + rank)
    grid = xa.build_param_grid(xa.GridConfig())
    n = len(grid.entries)
    eng = xa.Engine(dev.index)
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)
    da, db = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    counts = torch.zeros(n, dtype=torch.int32, device=dev)
    kpc = torch.zeros(n, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    mode = 1 if args.mode == "lanczos" else 0
    h, w = a.shape

    def step():
        eng.coarse_search_device(0, da.data_ptr(), w, h, db.data_ptr(), b.shape[1], b.shape[0], grid,
                                 MAX_POINTS, RATIO, mode, counts.data_ptr(), kpc.data_ptr(),
                                 stream.cuda_stream)

    torch.cuda.synchronize(dev)
    for _ in range(args.warmup):
        step()
    eng.check()
    launches_per_step = eng.last_launches()
    eng.set_profiling(not args.no_stage_events)
    stage_ms = {}
    kp_total = 0
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(dev.index) as clk:
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(k & 0xFF)
            starts[k].record(stream)
            step()
            ends[k].record(stream)
            for name, ms in eng.stage_times():
                stage_ms[name] = stage_ms.get(name, 0.0) + ms
            kp_total += int(kpc.sum().item())
        torch.cuda.synchronize(dev)
    barrier()
    eng.set_profiling(False)
    eng.check()
    total_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        # the one exchange of the path: gather every rank's per-view counts
        mine = counts.to(coll_dev)
        g = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(g, mine)
    ms_step = total_ms / args.steps
    value = world * n / (ms_step / 1e3)
    counters = eng.orb_counters(n + 1)
    work, stats = stage_work(xa, grid, w, h, counters)
    # dominant stage and its roofline
    per_step = {k: v / args.steps for k, v in stage_ms.items()}
    kernel_stages = {k: v for k, v in per_step.items() if k in work}
    if not kernel_stages:  # --no-stage-events: no per-stage timing, no roofline
        kernel_stages = {"none": 0.0}
        work = dict(work, none=("hbm", 0.0))
    dom = max(kernel_stages, key=kernel_stages.get)
    kind, amount = work[dom]
    peak, unit, src = peak_for(kind, sms, mhz, pk)
    sec = kernel_stages[dom] / 1e3
    achieved = amount / sec / (1e9 if unit == "GB/s" else 1e12) if sec > 0 else 0.0
    traffic = None
    try:  # DRAM bytes per launch of this stage from the committed ncu capture
        traffic = json.loads((ROOT / "profiles" / "traffic.json").read_text()).get(dom)
    except Exception:
        pass
    roof = {"bound": kind, "kernel": dom, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": achieved / peak, "traffic": traffic, "peak_source": src,
            "work_per_launch": amount, "ms_per_launch": kernel_stages[dom],
            "traffic_source": "profiles/traffic.json (ncu --set full, dram read+write bytes)"}
    if dom == "warp" and sec > 0:
        # the bound that actually binds the Lanczos taps (ncu r01: shared pipe ~66% busy over
        # the whole launch): every in-content output pixel reads its 64 taps (4 B each) from the
        # staged footprint; peak = 128 B/clk/SM of shared-memory bandwidth
        smem_peak = 128.0 * sms * mhz * 1e6 / 1e12
        smem_ach = 256.0 * stats["lanczos_px"] / sec / 1e12
        roof["shared_memory"] = {"achieved": smem_ach, "peak": smem_peak, "unit": "TB/s",
                                 "frac": smem_ach / smem_peak,
                                 "work": "64 taps x 4 B per in-content output px (lanczos_px)",
                                 "peak_source": f"128 B/clk/SM x {sms} SMs x {mhz:.0f} MHz"}
    stage_roof = {}
    for k, (kd, amt) in work.items():
        if k in per_step and per_step[k] > 0:
            pkk, un, _ = peak_for(kd, sms, mhz, pk)
            ach = amt / (per_step[k] / 1e3) / (1e9 if un == "GB/s" else 1e12)
            stage_roof[k] = {"ms": round(per_step[k], 4), "bound": kd, "achieved": round(ach, 3),
                             "unit": un, "frac": round(ach / pkk, 4)}

    # e2e through the public host API with pinned host buffers
    pa = torch.from_numpy(a).pin_memory()
    pb = torch.from_numpy(b).pin_memory()
    from paper_2503_03479_b200 import _lib
    import ctypes as C
    params = xa.api._params_array(grid)
    hc = np.zeros(n, np.int32)
    hk = np.zeros(n, np.int32)
    best = C.c_int32()

    def e2e_step():
        rc = _lib.lib().xa_coarse_search(eng.handle, 0, C.c_void_p(pa.data_ptr()), w, h,
                                         C.c_void_p(pb.data_ptr()), b.shape[1], b.shape[0], params, n,
                                         MAX_POINTS, RATIO, mode, hc.ctypes.data_as(C.c_void_p),
                                         hk.ctypes.data_as(C.c_void_p), C.byref(best))
        assert rc == 0, _lib.lib().xa_last_error()

    for _ in range(2):
        e2e_step()
    barrier()
    e2e_times = []
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(k & 0xFF)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        e2e_step()
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = sum(e2e_times)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_s], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = world * n * args.steps / e2e_s
    assert np.array_equal(hc, counts.cpu().numpy()), "e2e and device paths disagree"

    secondary = None
    if not args.no_secondary:
        secondary = {"config4_hamming": hamming_secondary(xa, eng, torch, dev, stream, pk, sms, mhz),
                     "config3_views": views_secondary(xa, eng, torch, dev, stream, pk, sms, mhz),
                     "fine_l2_ratio": l2_secondary(xa, eng, torch, dev, stream, pk, sms, mhz),
                     "fine_stage": fine_secondary(xa, eng, a, b, with_cpu=not args.no_cpu_baseline),
                     "asift_baseline": asift_secondary(xa, eng, a, b, with_cpu=not args.no_cpu_baseline),
                     "synth_warp_case": synth_secondary(xa, eng, a, with_cpu=not args.no_cpu_baseline)}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, info = cpu_baseline_run(np.array([p.as_tuple() for p in grid.entries]), a, b,
                                   os.cpu_count() or 1)
        cpu = {"value": v, "unit": "views/s", **info}
    if rank != 0:
        return
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": "views/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "views_per_step": n * world, "warp_mode": args.mode,
                   "l2": "flushed between steps (256 MiB write, untimed)",
                   "parallelism": f"weak: one pair per rank x {world}, views batched per launch",
                   "keypoints_per_s": kp_total * world / (total_ms / 1e3),
                   "hamming_cmp_per_s": stats["comparisons"] * world / (ms_step / 1e3)},
        "e2e": {"value": e2e_value, "unit": "views/s", "h2d_bytes_per_step": int(a.nbytes + b.nbytes),
                "d2h_bytes_per_step": int(2 * n * 4 + 4)},
        "roofline": roof,
        "stages": stage_roof,
        "stage_ms": {k: round(v, 4) for k, v in per_step.items()},
        "stats": {k: (round(v) if isinstance(v, float) else v) for k, v in stats.items()},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
        "cpu_baseline": cpu,
        "secondary": secondary,
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
