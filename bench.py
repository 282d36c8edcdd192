"""Benchmark of the DDF path-tracing hot path on B200 (contract: see DESIGN.md).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

A step is one full render (render.render_path) of the chosen BASELINE config
with inputs (weights, camera, RNG seed state) resident on the device; under
torchrun each rank renders its 64x64 tiles and the film is summed over NCCL.
Prints ONE JSON line on rank 0.  ``--impl reference`` times the reference
algorithm's CPU implementation (the float64 numpy oracle port, all host
threads) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_CONFIG = "c4"


def tensor_peak(prec, widths_list, long_step):
    """Roofline denominator for the MLP engine that `prec` selects.

    bf16: MEASURED_PEAKS.json's bf16 figure (sustained for kernels inside a
    long step, burst otherwise).  fp32 on networks <= 256 wide runs 3xTF32 on
    tcgen05: TF32 issues at half the bf16 rate (B200_PROFILING / guide table:
    1.13 vs 2.25 PF/s) and each product costs 3 MMAs, so the ceiling for
    algorithmic fp32 FLOPs is bf16 / 6.  fp32_simt (and fp32 on wider
    networks) is the FFMA pipe: 148 SMs x 128 FMA/clk x 2 x max SM clock."""
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    key = "bf16_tflops_sustained" if long_step else "bf16_tflops"
    bf16 = float(peaks[key]) if key in peaks else (1400.0 if long_step else 1590.0)
    src = ("MEASURED_PEAKS.json " + key) if key in peaks else "fallback " + ("sustained 1.4" if long_step else "burst 1.59") + " PF/s"
    x3 = prec == "fp32" and all(max(w[1:-1]) <= 256 and w[0] <= 96 and len(w) >= 3 for w in widths_list)
    if prec == "bf16":
        return bf16, src, "tensor"
    if x3:
        return bf16 / 6.0, src + " / 6 (3xTF32: tf32 at half the bf16 rate, 3 MMAs per product)", "tensor"
    mhz = float(peaks.get("sm_max_mhz", 1965.0))
    return 148 * 128 * 2 * mhz * 1e6 / 1e12, "FFMA pipe: 148 SMs x 128 FMA/clk x 2 x %.0f MHz" % mhz, "fma"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=["c1", "c2", "c3", "c4", "c5", "udf", "bvh", "march", "modes"])
    ap.add_argument("--precision", default=None, choices=[None, "fp32", "bf16", "fp32_simt"])
    ap.add_argument("--cpu-baseline", type=int, default=1, help="time the oracle port on rank 0 at N=1")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--tile-balance", default="rr", choices=["rr", "pilot"],
                    help="N>1: 64x64 tiles round-robin (config 4's rule, default) or by a measured spp=1 pilot "
                         "(LPT, every rank pilots its share)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only to exercise the multi-rank logic with several ranks on one GPU")
    return ap.parse_args()


# ----------------------------------------------------------------- CPU side
def oracle_field(name):
    from oracle import cpu_ddf as O
    from paper_2306_16142_b200 import configs as C
    nets = [O.Net(m.widths, m.v, m.g, m.b) for m in C.models(name)]
    w = C.WORKLOADS[name]
    if w.get("scene"):
        centers, scale, albedos = C.scene_layout()
        return O.Field(nets, C.CFG_DELTA, bounds=C.SCENE_BOX, centers=centers, scale=scale, albedos=albedos)
    return O.Field(nets, C.delta(name), bounds=C.UNIT_BOX)


def cpu_sample_bands(name):
    """Bounded CPU sample: pixel-row bands spread over the film at spp = 1
    (the stream prefix of sample 0), sized for ~10-30 s on 8 cores."""
    from paper_2306_16142_b200 import configs as C
    w = C.WORKLOADS[name]
    W, H = w["W"], w["H"]
    if name == "c2":
        return [(0, W * H)], w["spp"], "full render (128x128, 4 spp)"
    rows_total = {"c3": 32, "c4": 8, "c5": 16, "march": 8}[name]
    nb = 8
    per = max(1, rows_total // nb)
    bands = []
    for b in range(nb):
        y0 = int((b + 0.5) * H / nb) - per // 2
        bands.append((y0 * W, (y0 + per) * W))
    return bands, 1, f"{nb} bands x {per} rows x {W} px at spp=1 (stream prefix of sample 0)"


def cpu_render_sample(name):
    """One timed CPU step: (path samples, seconds)."""
    from oracle import cpu_ddf as O
    from paper_2306_16142_b200 import configs as C
    w = C.WORKLOADS[name]
    fld = oracle_field(name)
    cam = O.Cam((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), vfov=np.pi / 4, width=w["W"], height=w["H"])
    bands, spp, _ = cpu_sample_bands(name)
    cfg = O.PathConfig(spp=spp, bounces=w["bounces"], albedo=0.7, env=1.0, seed=C.RENDER_SEED,
                       rr_start=w.get("rr_start", -1))
    t0 = time.perf_counter()
    n = 0
    per_band = []
    for a, b in bands:
        tb = time.perf_counter()
        O.render_path(fld, cam, cfg, pix_range=(a, b))
        n += (b - a) * spp
        per_band.append((b - a) * spp / (time.perf_counter() - tb))
    cpu_render_sample.band_rates = per_band
    return n, time.perf_counter() - t0


def cpu_cores():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        nthr = max([i.get("num_threads", 1) for i in info] or [1])
    except Exception:
        nthr = os.cpu_count()
    return int(nthr)


def cpu_baseline(name, runs=1):
    _, _, desc = cpu_sample_bands(name)
    cpu_render_sample(name) if name != "c2" else None   # warm-up (BLAS threads, page-in)
    vals = []
    for _ in range(runs):
        n, s = cpu_render_sample(name)
        vals.append(n / s)
    out = {"value": statistics.median(vals), "unit": "path_samples/s", "cores": cpu_cores(), "kind": "port",
           "sample": desc + "; float64 numpy oracle (oracle/cpu_ddf.py), OpenBLAS threads"}
    rates = getattr(cpu_render_sample, "band_rates", [])
    if len(rates) > 1:   # sampling error of the band sample: spread of the per-band rates
        out["band_rate_rel_stderr"] = float(np.std(rates, ddof=1) / np.mean(rates) / np.sqrt(len(rates)))
    return out


# ----------------------------------------------------------------- config 1: query batch
def cpu_queries(args, reference_line=False):
    """Config 1 on the CPU: NeuralField.query_batch of the oracle (f64) on the
    full 65,536-ray batch, all OpenBLAS threads."""
    from oracle import cpu_ddf as O
    from paper_2306_16142_b200 import configs as C
    w = C.WORKLOADS["c1"]
    m = C.models("c1")[0]
    f = O.Field([O.Net(m.widths, m.v, m.g, m.b)], C.CFG_DELTA, bounds=C.UNIT_BOX)
    o, d = C.query_rays(w["n"], 0)
    f.query(o, d)
    reps = max(1, args.steps) if reference_line else 5
    t0 = time.perf_counter()
    for _ in range(reps):
        f.query(o, d)
    s = (time.perf_counter() - t0) / reps
    v = w["n"] / s
    base = {"value": v, "unit": "queries/s", "cores": cpu_cores(), "kind": "port",
            "sample": "full 65,536-ray batch, oracle query (field.py:248-258 restated), float64"}
    if not reference_line:
        return base
    return {"impl": "reference", "metric": "ddf_queries_per_s", "value": v, "unit": "queries/s", "n_gpus": args.gpus,
            "steps": reps, "warmup": 1, "ms_per_step": 1e3 * s, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": {"workload": "c1", "n": w["n"]},
            "cpu_baseline": base, "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0,
                                          "d2h_bytes_per_step": 0}}


def bench_queries(args, rank, world, local):
    """Config 1: one step = NeuralField.query_batch of 65,536 rays (5->4x128->1,
    fp32) through ddf_query, inputs resident on the device (value) and from
    pinned host arrays with results read back (e2e)."""
    import ctypes

    import torch
    from paper_2306_16142_b200 import _lib
    from paper_2306_16142_b200 import configs as C
    w = C.WORKLOADS["c1"]
    prec = args.precision or w["precision"]
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    f = C.build_field("c1", precision=prec)
    o, d = C.query_rays(w["n"], 0)
    n = w["n"]
    od, dd = torch.from_numpy(o).cuda(), torch.from_numpy(d).cuda()
    t = torch.empty(n, dtype=torch.float64, device="cuda")
    pred = torch.empty(n, dtype=torch.float64, device="cuda")
    hit = torch.empty(n, dtype=torch.uint8, device="cuda")
    L = _lib.lib()
    st = torch.cuda.current_stream()
    P = lambda x: ctypes.c_void_p(x.data_ptr())  # noqa: E731

    def step():
        _lib.check(L.ddf_query(f.handle, P(od), P(dd), n, P(t), P(hit), P(pred), None,
                               ctypes.c_void_p(st.cuda_stream)))
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    # Each step is one launch of tens of microseconds, so the steps are
    # enqueued without a host synchronize between them: the L2 flush ahead of
    # a step (a 256 MB write, ~40 us) runs while the host enqueues that step,
    # and the step's own CUDA events bracket the kernel alone.  With a
    # synchronize before every step the events also counted the host's launch
    # latency on an idle GPU (~10-15 us of the former 0.11 ms).
    evs = []
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            step()
            e1.record(st)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        clk.top_up(step)
    times = [a.elapsed_time(b) for a, b in evs]
    ms = float(np.mean(times))
    # e2e through the public protocol call (numpy in, numpy out); the call
    # takes well under a millisecond, so the mean is over at least 20 calls
    for _ in range(3):
        f.query_raw(o, d)
    te = []
    for _ in range(max(args.steps, 20)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f.query_raw(o, d)
        te.append(time.perf_counter() - t0)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    F = C.mlp_flops(w["widths"])
    ach = F * n / (ms / 1e3) / 1e12
    peak, peak_src, bound = tensor_peak(prec, [w["widths"]], False)
    out = {"metric": "ddf_queries_per_s", "value": n / (ms / 1e3), "unit": "queries/s", "n_gpus": world,
           "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": prec, "data": "synthetic",
           "config": {"workload": "c1", "n": n, "widths": list(w["widths"]), "precision": prec,
                      "l2": "flushed (256 MB write) before every timed step",
                      "timing": "CUDA events around each step, steps enqueued back to back (no host sync between)"},
           "roofline": {"bound": bound, "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                        "traffic": None, "kernel": "fused DDF-MLP query (65,536 rows = 3.5 tiles per SM)",
                        "peak_source": peak_src,
                        "frac_of_bf16_peak": ach / float(peaks.get("bf16_tflops", 1590.0))},
           "cpu_baseline": cpu_queries(args),
           "e2e": {"value": n / float(np.mean(te)), "unit": "queries/s", "h2d_bytes_per_step": 2 * n * 24,
                   "d2h_bytes_per_step": n * (8 + 8 + 1 + 4)},
           "gpu_launches": args.steps, "clocks": clk.summary()}
    # 65,536 rays are launch-latency bound; the large-N sweep
    # shows the engines' throughput (both precisions, same rays tiled)
    sweep = []
    for prc in ("fp32", "bf16"):
        fs = f if prc == prec else C.build_field("c1", precision=prc)
        for big in (1 << 20, 1 << 22, 1 << 24):
            reps = -(-big // n)
            ob, db = od.repeat(reps, 1)[:big].contiguous(), dd.repeat(reps, 1)[:big].contiguous()
            tb = torch.empty(big, dtype=torch.float64, device="cuda")
            hb = torch.empty(big, dtype=torch.uint8, device="cuda")
            call = lambda: _lib.check(L.ddf_query(fs.handle, P(ob), P(db), big, P(tb), P(hb), None, None,  # noqa: E731
                                                  ctypes.c_void_p(st.cuda_stream)))
            call()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(3):
                call()
            e1.record(st)
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 3
            sweep.append({"precision": prc, "rows": big, "ms": t, "queries_per_s": big / (t / 1e3),
                          "tflops": F * big / (t / 1e3) / 1e12})
    out["sweep"] = sweep
    out["sweep_note"] = ("5->4x128->1 on the four-slot (quad) engine: N = 128 MMAs are full rate, the bound is the "
                         "per-slot hand-off between epilogue and MMAs and the per-ray f64 angle trigonometry "
                         "(DESIGN.md section 3); fp32 runs 3xTF32 on tcgen05 (ceiling bf16 / 6)")
    if rank == 0:
        print(json.dumps(out))


# ----------------------------------------------------------------- UDF grid
UDF_RES, UDF_DIRS = 64, 512


def cpu_udf(args, reference_line=False):
    """recon.udf_grid on the CPU (oracle port, float64): a bounded sample of
    the grid's vertices (every 512th) with the full 512 directions + polish."""
    from oracle import cpu_ddf as O
    from paper_2306_16142_b200 import configs as C
    m = C.models("c1")[0]
    f = O.Field([O.Net(m.widths, m.v, m.g, m.b)], C.CFG_DELTA, bounds=C.UNIT_BOX)
    pts = O.grid_points(C.UNIT_BOX, UDF_RES)[::512]
    O.udf_many(f, pts[:4], UDF_DIRS)
    reps = max(1, args.steps) if reference_line else 1
    t0 = time.perf_counter()
    for _ in range(reps):
        O.udf_many(f, pts, UDF_DIRS)
    s = (time.perf_counter() - t0) / reps
    v = len(pts) / s
    desc = f"{len(pts)} of the {UDF_RES}^3 grid vertices (every 512th), {UDF_DIRS} dirs + polish, float64 oracle"
    base = {"value": v, "unit": "udf_points/s", "cores": cpu_cores(), "kind": "port", "sample": desc}
    if not reference_line:
        return base
    return {"impl": "reference", "metric": "udf_points_per_s", "value": v, "unit": "udf_points/s",
            "n_gpus": args.gpus, "steps": reps, "warmup": 1, "ms_per_step": 1e3 * s, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "udf", "resolution": UDF_RES, "n_dirs": UDF_DIRS, "sample": desc},
            "cpu_baseline": base, "e2e": {"value": v, "unit": "udf_points/s", "h2d_bytes_per_step": 0,
                                          "d2h_bytes_per_step": 0}}


def bench_udf(args, rank, world, local):
    """recon.udf_grid (recon.py:61-81) at 64^3 vertices x 512 directions +
    golden-section polish on the config-1 network; one step = one grid."""
    import ctypes

    import torch
    from paper_2306_16142_b200 import _lib
    from paper_2306_16142_b200 import configs as C
    from paper_2306_16142_b200 import udf as U
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    prec = args.precision or "bf16"
    f = C.build_field("c1", precision=prec)
    n = UDF_RES ** 3
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    box = (ctypes.c_double * 6)(*np.asarray(C.UNIT_BOX).reshape(-1))
    L = _lib.lib()
    st = torch.cuda.current_stream()

    def step():
        _lib.check(L.ddf_udf_grid(f.handle, box, UDF_RES, UDF_DIRS, 1, ctypes.c_void_p(out.data_ptr()),
                                  ctypes.c_void_p(st.cuda_stream)))
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    found = int(torch.isfinite(out).sum())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    times = []
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            step()
            e1.record(st)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        clk.top_up(step)
    ms = float(np.mean(times))
    te = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        U.udf_grid(f, resolution=UDF_RES, n_dirs=UDF_DIRS, bounds=C.UNIT_BOX)
        te.append(time.perf_counter() - t0)
    queries = n * UDF_DIRS + found * 2 * 2 * 13 * 2        # scan rows + polish probe rows (field.py:456-481)
    F = C.mlp_flops(C.WORKLOADS["c1"]["widths"])
    ach = F * queries / (ms / 1e3) / 1e12
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = float(peaks.get("bf16_tflops", 1590.0))
    n_scan = -(-n // ((1 << 25) // UDF_DIRS))
    # grid points, scan + argmin per chunk, compaction (1, single pass) + count, init, 4 x (begin, 13 probes, 12 steps, end), scatter
    launches = 1 + 2 * n_scan + 1 + 1 + 1 + 4 * 27 + 1
    res = {"metric": "udf_points_per_s", "value": n / (ms / 1e3), "unit": "udf_points/s", "n_gpus": world,
           "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": prec, "data": "synthetic",
           "config": {"workload": "udf", "resolution": UDF_RES, "n_dirs": UDF_DIRS, "polish": True,
                      "widths": list(C.WORKLOADS["c1"]["widths"]), "precision": prec,
                      "l2": "flushed (256 MB write) between timed steps"},
           "ddf_queries_per_s": queries / (ms / 1e3), "found_points": found,
           "roofline": {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                        "traffic": None, "kernel": "fused DDF-MLP (direction scan + polish probes), whole step"},
           "cpu_baseline": cpu_udf(args) if args.cpu_baseline else None,
           "e2e": {"value": n / float(np.mean(te)), "unit": "udf_points/s", "h2d_bytes_per_step": 48,
                   "d2h_bytes_per_step": 8 * n},
           "gpu_launches": args.steps * launches, "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(res))


# ----------------------------------------------------------------- BVH mesh render
BVH_MESH = "blob4"     # the reference's meshes.blob(4, 0): 5,120 triangles (tests/golden/reference_meshes.npz)


def reference_mesh(key=BVH_MESH):
    """(vertices, faces) of one of the reference's procedural meshes, as
    tests/golden/make_golden.py stored them."""
    z = np.load(os.path.join(ROOT, "tests", "golden", "reference_meshes.npz"))
    return z[f"{key}_v"], z[f"{key}_f"]


def cpu_bvh(args, reference_line=False):
    """render_path over the exact mesh field on the CPU: the oracle's float64
    linear scan (BruteForceField semantics) on a bounded band sample."""
    from oracle import cpu_ddf as O
    from paper_2306_16142_b200 import configs as C
    f = O.MeshField(*reference_mesh())
    w = C.WORKLOADS["c3"]
    cam = O.Cam((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), vfov=np.pi / 4, width=w["W"], height=w["H"])
    cfg = O.PathConfig(spp=1, bounces=w["bounces"], albedo=0.7, env=1.0, seed=C.RENDER_SEED)
    rows = [w["H"] // 2 + k for k in (-64, 0, 64)]
    O.render_path(f, cam, cfg, pix_range=(rows[0] * w["W"], rows[0] * w["W"] + 16))
    t0 = time.perf_counter()
    n = 0
    for r in rows:
        O.render_path(f, cam, cfg, pix_range=(r * w["W"], (r + 1) * w["W"]))
        n += w["W"]
    s = time.perf_counter() - t0
    v = n / s
    desc = f"3 pixel rows x {w['W']} px at spp=1 of the c3 camera, 5,120-triangle blob, float64 linear scan"
    base = {"value": v, "unit": "path_samples/s", "cores": cpu_cores(), "kind": "port", "sample": desc}
    if not reference_line:
        return base
    return {"impl": "reference", "metric": "path_samples_per_s", "value": v, "unit": "path_samples/s",
            "n_gpus": args.gpus, "steps": 1, "warmup": 1, "ms_per_step": 1e3 * s, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "bvh", "sample": desc}, "cpu_baseline": base,
            "e2e": {"value": v, "unit": "path_samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def bench_bvh(args, rank, world, local):
    """render.render_path with the exact mesh backend (OracleField over a BVH)
    at config 3's film, spp and bounces: the BVH side of the paper's
    DDF-vs-BVH render timing (Fig. 5)."""
    import torch
    from paper_2306_16142_b200 import configs as C
    from paper_2306_16142_b200 import render as R
    from paper_2306_16142_b200.mesh import CudaMeshField
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    fld = CudaMeshField(reference_mesh())
    cam = C.camera("c3")
    cfg = C.render_config("c3")
    n_pix = cam.width * cam.height
    accum = torch.empty(n_pix, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(max(3, args.warmup)):
        R.render_path_device(fld, cam, cfg, accum=accum, stream=stream)
    torch.cuda.synchronize()
    times = []
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _, st = R.render_path_device(fld, cam, cfg, accum=accum, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        clk.top_up(lambda: R.render_path_device(fld, cam, cfg, accum=accum, stream=stream))
    ms = float(np.mean(times))
    cfg.profile = 1
    _, prof = R.render_path_device(fld, cam, cfg, accum=accum, stream=stream)
    cfg.profile = 0
    te = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        R.render_path(fld, cam, cfg)
        te.append(time.perf_counter() - t0)
    samples = n_pix * cfg.spp
    res = {"metric": "path_samples_per_s", "value": samples / (ms / 1e3), "unit": "path_samples/s", "n_gpus": world,
           "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": "bvh", "mesh": "blob(4, 0)", "triangles": int(len(reference_mesh()[1])), "W": cam.width,
                      "H": cam.height, "spp": cfg.spp, "bounces": cfg.bounces,
                      "l2": "flushed (256 MB write) between timed steps"},
           "roofline": {"bound": "fp64", "achieved": None, "peak": None, "unit": None, "frac": None, "traffic": None,
                        "kernel": "BVH traversal (f64 Moller-Trumbore, one thread per ray)",
                        "trace_ms": prof["ms_forward"], "normal_ms": prof["ms_gradient"],
                        "compaction_ms": prof["ms_compact"], "other_ms": prof["ms_other"]},
           "cpu_baseline": cpu_bvh(args) if args.cpu_baseline else None,
           "e2e": {"value": samples / float(np.mean(te)), "unit": "path_samples/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 8 * n_pix},
           "gpu_launches": int(st["kernel_launches"]) * args.steps, "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(res))


# ----------------------------------------------------------------- single-bounce modes
def cpu_modes(args, reference_line=False):
    """render_depth / normal / shaded of the oracle (float64) on pixel-row bands."""
    from oracle import cpu_ddf as O
    W, H = 1920, 1080
    f = oracle_field("c4")
    cam = O.Cam((0.0, 0.0, 3.0), (0.0, 0.0, 0.0), vfov=np.pi / 4, width=W, height=H)
    bands = [np.arange((y * H) // 8 * W, ((y * H) // 8 + 1) * W) for y in range(8)]
    pix = np.concatenate(bands)
    t0 = time.perf_counter()
    for mode in ("depth", "normal", "shaded"):
        O.render_mode(f, cam, mode, pixels=pix)
    s = time.perf_counter() - t0
    v = 3 * len(pix) / s
    desc = f"8 pixel rows x {W} px of the 1920x1080 film per mode (depth, normal, shaded), c4 network, float64 oracle"
    base = {"value": v, "unit": "pixels/s", "cores": cpu_cores(), "kind": "port", "sample": desc}
    if not reference_line:
        return base
    return {"impl": "reference", "metric": "mode_pixels_per_s", "value": v, "unit": "pixels/s", "n_gpus": args.gpus,
            "steps": 1, "warmup": 0, "ms_per_step": 1e3 * s, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": {"workload": "modes", "sample": desc},
            "cpu_baseline": base, "e2e": {"value": v, "unit": "pixels/s", "h2d_bytes_per_step": 0,
                                          "d2h_bytes_per_step": 0}}


def bench_modes(args, rank, world, local):
    """render_depth / render_normal / render_shaded (render.py:144-184) at
    1920x1080 on the c4 network (the paper's Fig. 6 t-values / normal map /
    ray-traced), each one device call (ddf_render_mode); the same three over
    the exact BVH mesh (Fig. 5's BVH side).  One step = the three DDF modes."""
    import torch
    from paper_2306_16142_b200 import configs as C
    from paper_2306_16142_b200 import render as R
    from paper_2306_16142_b200.mesh import CudaMeshField
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    W, H = 1920, 1080
    prec = args.precision or "bf16"
    f = C.build_field("c4", precision=prec)
    mesh = CudaMeshField(reference_mesh("blob4"))
    cam = R.Camera(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), vfov=np.pi / 4, width=W, height=H)
    modes = ("depth", "normal", "shaded")

    bufs = {m: torch.empty(W * H * (1 if m == "depth" else 3), dtype=torch.float64, device="cuda") for m in modes}

    def timed(backend, mode, reps):
        cfg = R.RenderConfig(mode=mode)
        R.render_mode_device(backend, cam, cfg, mode, out=bufs[mode], to_host=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            R.render_mode_device(backend, cam, cfg, mode, out=bufs[mode], to_host=False)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(max(3, args.warmup)):
        for m in modes:
            R.render_mode_device(f, cam, R.RenderConfig(mode=m), m)
    per = {}
    with ClockSampler(dev) as clk:
        for m in modes:
            flush.zero_()
            per[m] = timed(f, m, args.steps)
        clk.top_up(lambda: [R.render_mode_device(f, cam, R.RenderConfig(mode=m), m) for m in modes])
    bvh = {m: timed(mesh, m, args.steps) for m in modes}
    ms = sum(per.values())
    te = []   # e2e: the public calls, image copied to the host
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for m in modes:
            R.render(f, cam, R.RenderConfig(mode=m))
        te.append(time.perf_counter() - t0)
    F = C.mlp_flops(C.WORKLOADS["c4"]["widths"])
    res = {"metric": "mode_pixels_per_s", "value": 3 * W * H / (ms / 1e3), "unit": "pixels/s", "n_gpus": world,
           "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": prec, "data": "synthetic",
           "config": {"workload": "modes", "W": W, "H": H, "network": "c4 65->8x512->1", "precision": prec,
                      "note": "images resident on the device in value; e2e copies them to the host"},
           "ddf_ms": per, "bvh_ms": bvh, "bvh_mesh": "blob(4, 0), 5,120 triangles",
           "roofline": {"bound": "tensor", "achieved": None, "peak": None, "unit": "TFLOP/s", "frac": None,
                        "traffic": None, "kernel": "trace step + (normal, shaded) gradient pass per pixel",
                        "algorithmic_flops_per_step": F * W * H * 3 + 2 * F * W * H * 2},
           "cpu_baseline": cpu_modes(args) if args.cpu_baseline else None,
           "e2e": {"value": 3 * W * H / float(np.mean(te)), "unit": "pixels/s", "h2d_bytes_per_step": 3 * 120,
                   "d2h_bytes_per_step": W * H * 8 * 7},
           "gpu_launches": None, "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(res))


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs a moment to start: wait for its first row so the
            # sampler is live when the timed region begins
            t_end = time.perf_counter() + 3.0
            while not self.rows and time.perf_counter() < t_end:
                time.sleep(0.01)
            self.start = len(self.rows)
        except Exception:
            self.proc = None
        self.extended_s = 0.0
        return self

    def top_up(self, fn, min_samples=3, max_s=3.0):
        """A timed region shorter than the 100 ms sample period may see no
        sample: keep the same work running (untimed) until a few samples
        land, and say so in the summary."""
        import torch
        t0 = time.perf_counter()
        while self.proc and len(self.rows) - self.start < min_samples and time.perf_counter() - t0 < max_s:
            fn()
            torch.cuda.synchronize()
        self.extended_s = time.perf_counter() - t0 if len(self.rows) - self.start else 0.0

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = self.rows[getattr(self, "start", 0):] or self.rows
        sm = [float(r[0]) for r in rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            if len(r) >= 8:
                for nm, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(nm)
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
               "reasons": sorted(reasons), "samples": len(rows)}
        if self.extended_s > 0.05:
            out["note"] = ("timed region shorter than the 100 ms sample period: sampled while the same step "
                           "kept running untimed for %.2f s after it" % self.extended_s)
        return out


# ----------------------------------------------------------------- GPU side
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    name = args.config

    if args.impl == "reference" and name == "c1":
        if rank != 0:
            return
        print(json.dumps(cpu_queries(args, reference_line=True)))
        return
    if args.impl == "reference" and name == "modes":
        if rank == 0:
            print(json.dumps(cpu_modes(args, reference_line=True)))
        return
    if args.impl == "reference" and name == "bvh":
        if rank == 0:
            print(json.dumps(cpu_bvh(args, reference_line=True)))
        return
    if args.impl == "reference" and name == "udf":
        if rank == 0:
            print(json.dumps(cpu_udf(args, reference_line=True)))
        return
    if args.impl == "reference":
        if rank != 0:
            return
        from paper_2306_16142_b200 import configs as C
        w = C.WORKLOADS[name]
        _, _, desc = cpu_sample_bands(name)
        for _ in range(args.warmup):
            cpu_render_sample(name)
        tot_n, tot_s = 0, 0.0
        for _ in range(args.steps):
            n, s = cpu_render_sample(name)
            tot_n += n
            tot_s += s
        v = tot_n / tot_s
        print(json.dumps({
            "impl": "reference", "metric": "path_samples_per_s", "value": v, "unit": "path_samples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "W": w["W"], "H": w["H"], "spp": w["spp"], "bounces": w["bounces"],
                       "sample": desc},
            "cpu_baseline": {"value": v, "unit": "path_samples/s", "cores": cpu_cores(), "kind": "port",
                             "sample": desc},
            "e2e": {"value": v, "unit": "path_samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    import torch
    import torch.distributed as dist
    from paper_2306_16142_b200 import configs as C
    from paper_2306_16142_b200 import render as R

    if name == "c1":
        return bench_queries(args, rank, world, local)
    if name == "udf":
        return bench_udf(args, rank, world, local)
    if name == "bvh":
        return bench_bvh(args, rank, world, local)
    if name == "modes":
        return bench_modes(args, rank, world, local)

    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    w = C.WORKLOADS[name]
    prec = args.precision or w["precision"]
    fld = C.build_field(name, precision=prec)
    cam = C.camera(name)
    cfg = C.render_config(name, rank=rank, world=world)
    from paper_2306_16142_b200.dist import balanced_owners_distributed, reduce_film, render_path_distributed
    pilot_s = None
    if world > 1 and args.tile_balance == "pilot":
        # setup, outside the timed region: every rank pilots its round-robin
        # share of the tiles at spp = 1, one exact sum of the cost vector, the
        # same LPT table on every rank (dist.balanced_owners_distributed)
        cfg.tile_owner, secs = balanced_owners_distributed(fld, cam, cfg, world)
        t = torch.tensor([secs], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        pilot_s = float(t.item())
    n_pix = cam.width * cam.height
    accum = torch.empty(n_pix, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    def step(profile=0):
        """One render of this rank's tiles plus the one collective: the film
        summed onto rank 0 (exact: every pixel has one non-zero term)."""
        cfg.profile = profile
        _, st = R.render_path_device(fld, cam, cfg, accum=accum, stream=stream)
        if world > 1:
            reduce_film(accum)
        return st

    for _ in range(max(3, args.warmup)):
        st = step()
    torch.cuda.synchronize()

    per_step = []
    launches = 0
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            flush.zero_()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            st = step()
            e1.record(stream)
            torch.cuda.synchronize()
            per_step.append(e0.elapsed_time(e1))
            launches += st["kernel_launches"]
        # rank-local work only (no collective: ranks may top up a different number of times)
        clk.top_up(lambda: R.render_path_device(fld, cam, cfg, accum=accum, stream=stream))
    ms_local = float(np.mean(per_step))
    t = torch.tensor([ms_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    samples_total = n_pix * cfg.spp
    value = samples_total / (ms / 1e3)

    # kernel-class breakdown (one profiled render; CUDA events on the launch stream)
    stp = step(profile=1)
    cfg.profile = 0
    torch.cuda.synchronize()
    models = C.models(name)
    F = sum(C.mlp_flops(m.widths) for m in models) if w.get("scene") else C.mlp_flops(models[0].widths)
    F_grad = 2 * C.mlp_flops(models[0].widths)   # one object's network per gradient row
    fwd_flops = F * stp["forward_rows"]
    # executed work: the separate gradient pass runs gradient_rows_executed
    # rows (2F each); fused trace+gradient rows add a backward chain (F) on
    # top of their forward, which forward_rows already counts
    grad_flops = F_grad * stp["gradient_rows_executed"]
    fused_flops = (F_grad // 2) * stp["fused_rows"]
    ref_flops = fwd_flops + F_grad * stp["gradient_rows"]
    mlp_ms = stp["ms_forward"] + stp["ms_gradient"] + stp["ms_fused"]
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    # burst peak for a kernel timed alone / in a short step, the sustained
    # (power-capped) figure for kernels timed inside a long step
    long_step = ms > 1000.0
    peak_tf, peak_src, bound = tensor_peak(prec, [m.widths for m in models], long_step)
    if long_step:
        peak_src += " (kernels inside a %.1f s step)" % (ms / 1e3)
    achieved_tf = (fwd_flops + grad_flops + fused_flops) / (mlp_ms / 1e3) / 1e12 if mlp_ms > 0 else 0.0
    roofline = {"bound": bound, "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": achieved_tf / peak_tf, "traffic": None,
                "kernel": "fused DDF-MLP (forward trace-step + input-gradient bounce)",
                "peak_source": peak_src,
                "frac_of_burst_peak": achieved_tf / tensor_peak(prec, [m.widths for m in models], False)[0],
                "frac_of_bf16_peak": achieved_tf / float(peaks.get("bf16_tflops", 1590.0)),
                "mlp_share_of_step": mlp_ms / stp["ms_total"] if stp["ms_total"] else None,
                "forward": {"rows": stp["forward_rows"] - stp["fused_rows"], "ms": stp["ms_forward"],
                            "launches": stp["forward_launches"],
                            "tflops": F * (stp["forward_rows"] - stp["fused_rows"]) / (stp["ms_forward"] / 1e3) / 1e12
                            if stp["ms_forward"] else None},
                "gradient": {"rows": stp["gradient_rows_executed"], "ms": stp["ms_gradient"],
                             "launches": stp["gradient_launches"],
                             "tflops": grad_flops / (stp["ms_gradient"] / 1e3) / 1e12 if stp["ms_gradient"] else None},
                "fused_trace_gradient": {
                    "rows": stp["fused_rows"], "ms": stp["ms_fused"], "launches": stp["fused_launches"],
                    "tflops": (F * stp["fused_rows"] + fused_flops) / (stp["ms_fused"] / 1e3) / 1e12
                    if stp["ms_fused"] else None,
                    "note": "bounce-ray march step 0 + the next bounce's normal gradient in one kernel where the "
                            "inputs coincide (SURVEY 8(d) fused normal reuse): forward F + backward F per row"},
                "compaction_ms": stp["ms_compact"], "other_ms": stp["ms_other"], "profiled_step_ms": stp["ms_total"]}
    # wavefront compaction against HBM: per compaction call the
    # flags are read once (single pass), or twice with the 4 B object ids when
    # bucketed (the scene's bounce stage), and 4 B are written per survivor;
    # the survivors are exactly the MLP rows
    import math
    lo_b, hi_b = np.asarray(C.SCENE_BOX if w.get("scene") else C.UNIT_BOX)
    diag = float(np.sqrt(((hi_b - lo_b) ** 2).sum()))
    max_steps = math.ceil(diag / (0.9 * C.delta(name))) + 4
    samples = int(stp["path_samples"])
    calls = max_steps * (1 + cfg.bounces) + cfg.bounces
    bucketed = cfg.bounces if w.get("scene") else 0
    cbytes = samples * (calls - bucketed) + (2 + 8) * samples * bucketed \
        + 4 * (stp["forward_rows"] + stp["gradient_rows"])
    hbm = float(peaks.get("hbm_gbs", 6540.5))
    if stp["ms_compact"]:
        gbps = cbytes / (stp["ms_compact"] / 1e3) / 1e9
        roofline["compaction"] = {"bound": "hbm", "ms": stp["ms_compact"], "bytes": cbytes, "achieved": gbps,
                                  "peak": hbm, "unit": "GB/s", "frac": gbps / hbm,
                                  "calls_per_wave": calls, "note": "launch-latency bound below ~8 M slots per call"}
    # the wavefront kernels against HBM: algorithmic bytes are
    # the path-state fields each kernel must read and write (structure of
    # arrays, f64; wavefront.cuh), minimum counts where a write depends on
    # the path's outcome
    P = samples
    alive_rows = int(sum(stp["bounce_alive_rows"]))
    rr_b = max(0, cfg.bounces - cfg.rr_start) if cfg.rr_start >= 0 else 0
    own = n_pix if world == 1 else int(stp["path_samples"]) // cfg.spp
    wave_bytes = {
        # pix 4 | o, d 48 | thr, rad 16 | alive 1 | u34 16 | t_acc, t_exit, t 24 | march, hit, gdone 3 | obj 4
        "camera_kernel": ("ms_camera", 116 * P, "per slot: pixel id in; o, d, throughput, radiance, trace state out"),
        # per slot: hit in, alive out; per bounce-alive row: list entry + hit in
        "after_kernels": ("ms_after", 2 * P + 5 * alive_rows, "after_primary (hit -> alive) + after_bounce (list, hit)"),
        # per slot and RR bounce: alive in; per surviving row: pixel id + throughput in, throughput out
        "roulette_kernel": ("ms_roulette", rr_b * P + 20 * alive_rows if rr_b else 0, "alive flags, survivors' throughput"),
        # per alive row: list 4 | o, d, g3 72 | t 8 | obj 4 | thr 8 | pix 4 in; thr 8 | o, d 48 | trace state 47 | want 1 out
        "bounce_kernel": ("ms_bounce", 204 * alive_rows, "normal, hit point, cosine bounce, slab test"),
        # per owned pixel: id 4, accumulator 8 in and out; per slot: radiance 8
        "film_kernel": ("ms_film", 20 * own * stp["waves"] + 8 * P, "accum += radiance in spp order"),
    }
    wf = {}
    for kname, (key, nbytes, what) in wave_bytes.items():
        t_ms = stp.get(key) or 0.0
        if t_ms > 0 and nbytes > 0:
            gbps = nbytes / (t_ms / 1e3) / 1e9
            wf[kname] = {"ms": t_ms, "bytes": int(nbytes), "achieved": gbps, "frac": gbps / hbm, "what": what}
    roofline["wavefront"] = {"bound": "hbm", "peak": hbm, "unit": "GB/s", "kernels": wf}

    # DRAM traffic per launch of the dominant kernel from the committed ncu
    # --set full capture of this workload (profiles/), next to the
    # algorithmic path-state bytes of that launch
    ncu_path = None
    for ver in ("r2_%s_ncu_v6", "r2_%s_ncu_v3", "r1_%s_ncu_v11"):
        cand = os.path.join(ROOT, "profiles", (ver % name) + ".json")
        if os.path.exists(cand):
            ncu_path = cand
            break
    if ncu_path:
        try:
            rec = json.load(open(ncu_path))
            key = "fused_launch" if "fused_launch" in rec else "gradient_launch"
            g = rec[key]
            kname = g.get("kernel", "mlp_kernel<GradOutOp>").split("(")[0].replace("void ", "")
            roofline["traffic"] = g["traffic_bytes"]
            roofline["traffic_source"] = ("ncu --set full, one %s launch of %.1f ms (%s): %.0f MB DRAM vs ~%.0f MB "
                                          "algorithmic path state; tensor pipe active %.1f%%" % (
                                              kname, g["duration_ms"], os.path.basename(ncu_path),
                                              g["traffic_bytes"] / 1e6, g["algorithmic_state_bytes_est"] / 1e6,
                                              g["tensor_pipe_active_pct_elapsed"]))
        except Exception:
            pass

    # end to end through the public API (render.render_path at N = 1,
    # dist.render_path_distributed at N > 1): each call allocates its own
    # accumulator, uploads the PCG64 jump tables and returns the (H, W, 3)
    # film on the host (rank 0)
    e2e = None
    if not args.no_e2e:
        ts = []
        for _ in range(args.steps):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            if world > 1:
                render_path_distributed(fld, cam, cfg, tile_owner=cfg.tile_owner)
            else:
                R.render_path(fld, cam, cfg)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        te = torch.tensor([float(np.mean(ts))], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": samples_total / te.item(), "unit": "path_samples/s",
               "h2d_bytes_per_step": 2 * (16 + 64 * 32) + 0,   # PCG64 jump tables (camera/config are kernel params)
               "d2h_bytes_per_step": n_pix * 8 + 160,
               "api": "render.render_path" if world == 1 else "dist.render_path_distributed"}

    cpu = None
    if rank == 0 and world == 1 and args.cpu_baseline:
        cpu = cpu_baseline(name)

    if rank == 0:
        out = {
            "metric": "path_samples_per_s", "value": value, "unit": "path_samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": prec, "data": "synthetic",
            "config": {"workload": name, "W": cam.width, "H": cam.height, "spp": cfg.spp, "bounces": cfg.bounces,
                       "widths": list(models[0].widths), "n_networks": len(models), "precision": prec,
                       "tiles": cfg.tile, "parallelism": f"tiles{world}" if world > 1 else "single",
                       "tile_assignment": (("pilot-balanced (LPT)" if cfg.tile_owner is not None else "round-robin")
                                           if world > 1 else None),
                       "collective": (f"film sum-reduce to rank 0 ({args.dist_backend.upper() if args.dist_backend != 'nccl' else 'NCCL'}), inside the step"
                                 if world > 1 else None),
                       "l2": "flushed (256 MB write) between timed steps"},
            "ddf_queries_per_s": stp["forward_rows"] / (ms / 1e3),
            "gradient_rows_per_s": stp["gradient_rows"] / (ms / 1e3),
            "flops_per_step": fwd_flops + grad_flops + fused_flops,
            "reference_equivalent_flops_per_step": ref_flops,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk.summary(),
        }
        if pilot_s is not None:
            out["pilot_setup_s"] = pilot_s
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
