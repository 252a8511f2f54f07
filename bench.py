#!/usr/bin/env python
"""Benchmark: ms per Sp-MART iteration and ray-voxel updates/s on the USPG
slice stack (BASELINE.json configs[1], "C2"), plus % of the HBM roofline.

A step is one MART iteration (one full sweep over every view and line) of all
S problems of the stack. `value` is measured on device-resident data with
CUDA events; `e2e` runs the same step through the C ABI with pinned host
buffers (projections + field H2D, field D2H inside the timed region).

    python bench.py [--gpus N --steps K --warmup W --config c2 --impl ours|reference]

Multi-GPU (torchrun, one rank per GPU): every rank reconstructs its own stack
of S slices (weak scaling; slices are independent problems, no collective on
the data path). Timing = max over ranks of the device time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "traffic.json")
FALLBACK_HBM = 6650.0


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU arm: the oracle restatement (pinned bit-exact to the reference library)
# ---------------------------------------------------------------------------
def cpu_run(wl, proj, sample_problems: int, sweeps: int, threads: int):
    """Run `sample_problems` slices x `sweeps` MART sweeps of the oracle with
    one slice per host thread; returns (updates/s, wall s, updates, problems)."""
    import oracle

    orc = oracle.Orc()
    spec = wl.spec
    volume = spec.mode.value == 1
    g = oracle.OrcGrid(spec.rings(), spec.ring_spacing, spec.slices(), spec.slice_height, volume,
                       None if spec.ring_counts is None else np.asarray(spec.ring_counts, np.uint32))
    src, det = wl.geom.first_view_rays()
    cache = orc.cache(g, src, det)
    th = wl.geom.thetas()
    caches = [cache] + [orc.cache(g, src, det) for _ in range(min(threads, sample_problems) - 1)]
    results = [None] * sample_problems

    def work(i, c):
        f, rep = c.reconstruct(th, proj[i].astype(np.float64), beta=wl.beta, tolerance=0, max_sweeps=sweeps)
        results[i] = rep["updates"]

    t0 = time.perf_counter()
    pending = list(range(sample_problems))
    lock = threading.Lock()

    def worker(c):
        while True:
            with lock:
                if not pending:
                    return
                i = pending.pop(0)
            work(i, c)

    ths = [threading.Thread(target=worker, args=(c,)) for c in caches]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    wall = time.perf_counter() - t0
    upd = int(sum(results))
    return upd / wall, wall, upd, len(caches)


def ref_lib_analogue(threads: int):
    """The unmodified reference library on the C2 reference analogue (one
    slice, one sweep): square_2d(512), flat panel — the closest config it can
    express."""
    import oracle

    if not os.path.exists(oracle.REF_SO):
        return None
    from paper_2208_12964_b200 import workloads
    wl = workloads.make("c2-ref", problems=1)
    ref = oracle.Ref()
    g = wl.geom
    rt = ref.tracer(512, False, g.source, g.detector_center, g.det_u, 1, g.spacing_u, 0.0, g.views, False, threads)
    rng = np.random.default_rng(1)
    truth = ref.phantom(512, False) * rng.uniform(0.5, 1.0)
    p = rt.project(truth)
    t0 = time.perf_counter()
    f, rep = rt.reconstruct(p, beta=0.05, tolerance=0, max_sweeps=1)
    wall = time.perf_counter() - t0
    # U from the trace counters: every non-skipped line's |active|
    upd = 0
    th = [v * (360.0 / g.views) for v in range(g.views)]
    for v in range(g.views):
        for line in range(g.det_u):
            if p[v, line] != 0:
                upd += rt.trace_line(line, th[v]).size
    return {"value": upd / rep["seconds"], "unit": "updates/s", "cores": 1, "kind": "reference",
            "sample": "oracle/_ref (unmodified reference) on c2-ref: square_2d(512), flat 512-det fan, 90 views, "
                      "1 slice x 1 sweep (reconstruct is single-threaded by design)",
            "seconds": rep["seconds"]}


def run_reference(args, rank, world):
    from paper_2208_12964_b200 import workloads

    if rank != 0:
        return
    wl = workloads.make(args.config, problems=args.problems)
    threads = max(1, os.cpu_count() or 1)
    S = wl.problems
    sample = min(S, 2 * threads)
    truth = workloads.phantom_fields(wl, sample)
    # projections: binary model of the same tracer, on the CPU oracle
    import oracle
    orc = oracle.Orc()
    spec = wl.spec
    g = oracle.OrcGrid(spec.rings(), spec.ring_spacing, spec.slices(), spec.slice_height,
                       spec.mode.value == 1, None if spec.ring_counts is None else spec.counts())
    src, det = wl.geom.first_view_rays()
    oc = orc.cache(g, src, det)
    th = wl.geom.thetas()
    proj = np.stack([oc.project(th, truth[i].astype(np.float32).astype(np.float64)) for i in range(sample)])
    proj = workloads.add_noise(wl, proj.astype(np.float32))
    vals = []
    for _ in range(args.warmup):
        cpu_run(wl, proj, sample, 1, threads)
    walls = []
    for _ in range(args.steps):
        v, wall, upd, used = cpu_run(wl, proj, sample, 1, threads)
        vals.append(v)
        walls.append(wall)
    value = float(np.median(vals))
    # one full iteration of the whole stack at this throughput
    ms_iter = 1e3 * float(np.median(walls)) * S / sample
    line = {
        "impl": "reference", "metric": metric_name(args.config), "value": value, "unit": "updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_iter,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded random-ellipse phantoms, binary projections, 1% Gaussian noise",
        "config": config_dict(wl, args),
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": used, "kind": "port",
                         "sample": f"{sample} of {S} slices x 1 sweep per step, one slice per host thread "
                                   f"(oracle C restatement, pinned bit-exact to the reference library; the "
                                   f"reference cannot express the verbatim config, SURVEY.md §0.1)"},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def mart_kernel_name(Sp, executor):
    """The MART kernel the library ran (uscg_tracer_info.executor)."""
    p = 1
    lim = int(os.environ.get("USCG_CHUNK_WIDTH", 32))
    while p * 2 <= lim and Sp % (p * 2) == 0:
        p *= 2
    if executor == 3:
        return f"mart_wave_kernel<{p}> (one persistent launch per reconstruct call; task = (view, {p}-problem chunk))"
    if executor == 2:
        return f"mart_level_kernel<{p}> (one launch per dependency level)"
    if executor == 1:
        return f"mart_sweep_kernel<{p}> (one cooperative launch per sweep)"
    return f"mart_flow_kernel<{p}> (one dataflow launch per reconstruct call)"


def metric_name(config):
    return f"ray-voxel updates/s per Sp-MART iteration ({config})"


def config_dict(wl, args):
    spec, geom = wl.spec, wl.geom
    return {"workload": args.config, "problems": wl.problems, "rings": spec.rings(),
            "sector_law": "reference 4(2k-1)" if spec.ring_counts is None else "round(2*pi*(i+0.5))",
            "cells_per_slice": spec.cells_per_slice(), "slices": spec.slices(), "views": geom.views,
            "detectors": [geom.det_u, geom.det_v], "detector": geom.detector.name.lower(), "beta": wl.beta,
            "iterations_per_reconstruction": wl.sweeps,
            "l2": "timed iterations run back to back in one reconstruct call; working set > L2 "
                  "(field + projections + schedule); 'isolated' repeats with L2 flushed per iteration",
            "parallelism": f"{wl.problems} independent slices per GPU (weak scaling)"}


# ---------------------------------------------------------------------------
# C5: coefficient generation, rotated reuse, USPG -> CG resampling
# ---------------------------------------------------------------------------
def bench_c5(args, rank, world, local):
    """BASELINE configs[4]. Three device-timed legs:
    (1) the first-view generator over the 1024x1024 panel (rays/s; device time
    reported by the library, count + scan + write + annotate); (2) rotated
    reuse: every (view, line) of 180 views served from the one-view record
    store, |active| + index checksum per line (lines/s; bytes 20*C + 12*L per
    view); (3) resampling a seeded U[0,1] 512-ring x 512-slice USPG volume to
    1024 x 1024 x 512 (8 B per output pixel). N > 1 ranks split detector rows,
    views and slices (strong scaling); the generator's one exchange assembles
    the full record store on every rank (dist.assemble_cache)."""
    import torch
    import torch.distributed as dist

    import paper_2208_12964_b200 as ub
    from paper_2208_12964_b200 import dist as udist
    from paper_2208_12964_b200 import uscg, workloads

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = workloads.make("c5")
    spec, geom = wl.spec, wl.geom
    ctx = ub.Context(local)
    # one stream for torch and the library: events time the launching stream
    # (the legacy default stream's handle is 0, which the ABI reads as "the
    # context's own stream")
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    L = ub.load()
    src, det = geom.first_view_rays()
    lines = geom.lines()
    rows = geom.det_v
    r0, r1 = rank * rows // world, (rank + 1) * rows // world
    mine = slice(r0 * geom.det_u, r1 * geom.det_u)

    # (1) generator on this rank's detector rows (1-view tracers; the record
    #     store is rebuilt every step)
    gen_ms = []
    recs = 0
    for k in range(args.warmup + args.steps):
        tr = ub.Tracer.from_rays(spec, src[mine], det[mine], 1, ctx=ctx)
        inf = tr.info()
        if k >= args.warmup:
            gen_ms.append(inf["generator_ms"])
        recs = inf["records"]
        tr.close()
    g_ms = float(np.mean(gen_ms))
    rays_mine = (r1 - r0) * geom.det_u

    # the full record store on every rank: one rank alone generates it; N
    # ranks exchange their row blocks (dist.assemble_cache: all-gather of the
    # counts and of the padded segments over NCCL)
    exchange_ms = 0.0
    if world > 1:
        local_tr = ub.Tracer.from_rays(spec, src[mine], det[mine], 1, ctx=ctx)
        part = local_tr.copy_cache(device=True)
        local_tr.close()
        torch.cuda.synchronize()
        dist.barrier()
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x0.record(stream)
        full = udist.assemble_cache(*part)
        x1.record(stream)
        torch.cuda.synchronize()
        exchange_ms = x0.elapsed_time(x1)
        tr = ub.Tracer.from_key_cache(spec, *full, geom.views, geom.view_angles, geom=geom, ctx=ctx)
        del full, part
    else:
        tr = ub.Tracer(geom, spec, False, ctx=ctx)
    # (2) rotated reuse over this rank's views
    inf = tr.info()
    v0, v1 = rank * geom.views // world, (rank + 1) * geom.views // world
    nv = v1 - v0
    counts_d = torch.empty(nv * lines, dtype=torch.int32, device="cuda")
    sums_d = torch.empty(nv * lines, dtype=torch.int64, device="cuda")

    def reuse():
        uscg._check(L.uscg_trace_checksums(tr.h, v0, nv, uscg.C.c_void_p(counts_d.data_ptr()),
                                           uscg.C.c_void_p(sums_d.data_ptr()), uscg.DEVICE_POINTERS))

    for _ in range(args.warmup):
        reuse()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ub.launch_count()
    e0.record(stream)
    for _ in range(args.steps):
        reuse()
    e1.record(stream)
    torch.cuda.synchronize()
    reuse_ms = e0.elapsed_time(e1) / args.steps
    chords = inf["records"] * nv  # chords traversed per pass (records x views)
    reuse_bytes = 20 * chords + 12 * nv * lines
    # parity spot check against the library's own per-line counts
    cnt_ref = tr.trace_counts()[v0:v1].reshape(-1)
    reuse_ok = bool(np.array_equal(counts_d.cpu().numpy().astype(np.uint32), cnt_ref))
    tr.close()

    # (3) resample this rank's slices of a seeded U[0,1] volume
    sl0, sl1 = rank * spec.slices() // world, (rank + 1) * spec.slices() // world
    sub = ub.GridSpec(spec.n, spec.ring_spacing, spec.slice_height, spec.mode, ring_counts=spec.ring_counts,
                      n_slices=sl1 - sl0)
    npix = 1024
    gen = torch.Generator(device="cuda")
    gen.manual_seed(12345 + rank)
    field_d = torch.rand(sub.cell_count(), dtype=torch.float32, device="cuda", generator=gen)
    img_d = torch.empty((sl1 - sl0, npix, npix), dtype=torch.float32, device="cuda")
    g_c, keep = sub._c()

    def resample():
        uscg._check(L.uscg_resample(ctx.h, uscg.C.byref(g_c), uscg.C.c_void_p(field_d.data_ptr()), 1, npix,
                                    uscg.C.c_void_p(img_d.data_ptr()), uscg.DEVICE_POINTERS))

    for _ in range(args.warmup):
        resample()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        resample()
    e1.record(stream)
    torch.cuda.synchronize()
    res_ms = e0.elapsed_time(e1) / args.steps
    # (4) volume image-quality scores of the resampled volume against a
    #     perturbed copy (mae / rmse / ssim per slice, shared ssim range as
    #     ssim_volume, metrics.cpp:170-199)
    test_d = img_d * 0.97 + 0.01
    nsl = sl1 - sl0
    m_mae, m_rmse, m_ssim = np.zeros(nsl), np.zeros(nsl), np.zeros(nsl)
    dp = uscg.C.POINTER(uscg.C.c_double)

    def metrics():
        uscg._check(L.uscg_image_metrics(ctx.h, uscg.C.c_void_p(img_d.data_ptr()),
                                         uscg.C.c_void_p(test_d.data_ptr()), nsl, npix, npix, 1, -1.0,
                                         m_mae.ctypes.data_as(dp), m_rmse.ctypes.data_as(dp),
                                         m_ssim.ctypes.data_as(dp), uscg.DEVICE_POINTERS))

    metrics()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        metrics()
    e1.record(stream)
    torch.cuda.synchronize()
    met_ms = e0.elapsed_time(e1) / args.steps
    launches = ub.launch_count() - launches0
    clk = clocks.stop()
    px = (sl1 - sl0) * npix * npix
    g_ms, reuse_ms, res_ms, met_ms, exchange_ms = udist.max_over_ranks(
        [g_ms, reuse_ms, res_ms, met_ms, exchange_ms], device="cuda")
    rays_all, recs_all = udist.sum_over_ranks([rays_mine, recs], device="cuda")

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    peak, peak_kind = hbm_peak()
    gen_bytes = 20 * recs_all + 4 * (lines + 1)
    reuse_bytes_all = reuse_bytes * world
    res_bytes = 8 * px * world

    def roof(bytes_, ms, kernel, model):
        a = bytes_ / (ms * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": a, "peak": peak, "unit": "GB/s", "frac": a / peak, "traffic": None,
                "peak_kind": peak_kind, "kernel": kernel, "bytes_model": model}

    cpu = None
    if not args.no_cpu and world == 1:
        import oracle

        orc = oracle.Orc()
        og = oracle.OrcGrid(spec.rings(), spec.ring_spacing, spec.slices(), spec.slice_height, True,
                            spec.ring_counts)
        pick = np.random.default_rng(5).choice(lines, 512, replace=False)
        t0 = time.perf_counter()
        oc = orc.cache(og, src[pick], det[pick])
        wall = time.perf_counter() - t0
        cpu = {"value": pick.size / wall, "unit": "rays/s", "cores": 1, "kind": "port",
               "sample": f"oracle C restatement of precompute_first_view on {pick.size} random rays of the panel "
                         f"({wall:.1f} s, {int(oc.offsets[-1])} records)"}
    value = rays_all / ((g_ms + exchange_ms) * 1e-3)  # generation + the exchange that assembles the store
    line = {
        "metric": "first-view generator rays/s (c5)", "value": value, "unit": "rays/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": g_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: BASELINE c5 geometry; seeded U[0,1] USPG volume for the resample",
        "config": {"workload": "c5", "rings": spec.rings(), "sector_law": "round(2*pi*(i+0.5))",
                   "slices": spec.slices(), "cells": spec.cell_count(), "detectors": [geom.det_u, geom.det_v],
                   "views": geom.views, "resample_pixels": [npix, npix, spec.slices()],
                   "l2": "working sets (11.6 GB record store, 1.7 + 2.1 GB volumes) exceed L2",
                   "parallelism": "rows / views / slices split across ranks"},
        "roofline": roof(gen_bytes, g_ms, "generate_bound_kernel + generate_slot_kernel + compact_records_kernel + annotate_kernel",
                         "20*records + 4*(lines+1) written (SURVEY.md §8(d))"),
        "generator": {"ms": g_ms, "exchange_ms": exchange_ms, "rays": rays_all, "records": recs_all,
                      "records_per_s": recs_all / ((g_ms + exchange_ms) * 1e-3)},
        "rotated_reuse": {"ms": reuse_ms, "views": geom.views, "lines_per_s": world * nv * lines / (reuse_ms * 1e-3),
                          "chords_per_s": world * chords / (reuse_ms * 1e-3), "counts_match_library": reuse_ok,
                          "roofline": roof(reuse_bytes_all, reuse_ms, "checksum_kernel<128>",
                                           "20*C + 12*L per view (SURVEY.md §8(d))")},
        "resample": {"ms": res_ms, "pixels": px * world, "pixels_per_s": px * world / (res_ms * 1e-3),
                     "roofline": roof(res_bytes, res_ms, "bin_map_kernel + map_resample_kernel",
                                      "8 B per output pixel (SURVEY.md §8(d))")},
        "metrics": {"ms": met_ms, "slices": nsl * world, "ssim_volume": float(m_ssim.mean()),
                    "rmse_volume": float(m_rmse.mean()), "pixels_per_s": px * world / (met_ms * 1e-3),
                    "roofline": roof(res_bytes, met_ms, "moments_kernel + ssim_kernel",
                                     "8 B per pixel pair read (two fp32 rasters; SURVEY.md §8(f) row 3)")},
        "cpu_baseline": cpu, "e2e": None, "gpu_launches": int(launches), "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# the paper's comparison: USPG vs Cartesian Siddon MART (proj/src/bench.cpp)
# ---------------------------------------------------------------------------
def bench_cmp(args, rank, world, local):
    """bench_compare (bench.cpp:24-88) with acceptance_9's configuration
    (acceptance.cpp:600-611: n 256, 101 detectors, spacing 0.05, 50 views,
    30 sweeps, beta 0.4) on the device: storage of the symmetry-compressed
    cache vs the stored Cartesian system for p = 10 / 50 / 100 views, and the
    time of the polar pipeline (cache build + sweeps) against Cartesian MART
    with Siddon on the fly (sweeps) and stored (precompute + sweeps). The
    reference's own CPU times for the same comparison are measured beside it.
    Rank 0 only (one problem; no sharding)."""
    import torch

    import paper_2208_12964_b200 as ub
    from paper_2208_12964_b200 import uscg, workloads

    if rank != 0:
        return
    torch.cuda.set_device(local)
    n, det, spacing, views, sweeps, beta = 256, 101, 0.05, 50, 30, 0.4
    spec = ub.GridSpec.square_2d(n)

    def geom_of(p):
        return ub.ScanGeometry(source=(-8, 0, 0), detector_center=(8, 0, 0), det_u=det, spacing_u=spacing, views=p)

    quarter = det % 2 == 1  # ScanGeometry::quarter_symmetric (scan.cpp:44-48): odd panel, on-axis source

    memory = []
    for p in (10, 50, 100):
        g = geom_of(p)
        tr = ub.Tracer(g, spec, quarter)
        inf = tr.info()
        cs = ub.CartesianSystem(spec, g, stored=True)
        cinf = cs.info()
        rows = p * det
        memory.append({"views": p, "polar_cache_bytes": inf["cache_bytes"],
                       "cartesian_stored_bytes": cinf["device_bytes"],
                       "ratio": cinf["device_bytes"] / inf["cache_bytes"],
                       "reference_layout": {"polar_cache_bytes": 24 * inf["records"] + 4 * (det + 1),
                                            "cartesian_stored_bytes": 8 * (rows + 1) + 12 * cinf["entries"]}})
        tr.close()
        cs.close()

    geom = geom_of(views)
    wl = workloads.make("c1-ref")  # seeded random-ellipse phantom generator (no Shepp-Logan table bundled)
    wl.spec = spec
    truth = workloads.phantom_fields(wl, 1)[0]
    tr0 = ub.Tracer(geom, spec, quarter)
    proj = ub.project_stack(tr0, truth[None, :].astype(np.float32))[0]
    tr0.close()
    cfg = ub.SolverConfig(beta=beta, tolerance=0, max_sweeps=sweeps)

    def polar():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tr = ub.Tracer(geom, spec, quarter)
        res = ub.reconstruct(ub.ProjectionSet(geom, proj.astype(np.float64)), spec, cfg, tr)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        tr.close()
        return wall, res.report.seconds

    def cartesian(stored):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cs = ub.CartesianSystem(spec, geom, stored=stored)
        field, sec = cs.reconstruct(proj, cfg)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        info = cs.info()
        cs.close()
        return wall, sec, info

    for _ in range(max(1, args.warmup)):
        polar(), cartesian(False), cartesian(True)
    reps = max(1, args.steps)
    pol = [polar() for _ in range(reps)]
    otf = [cartesian(False) for _ in range(reps)]
    sto = [cartesian(True) for _ in range(reps)]
    polar_s = float(np.median([w for w, _ in pol]))
    polar_sweeps_s = float(np.median([s for _, s in pol]))
    otf_sweeps_s = float(np.median([s for _, s, _ in otf]))
    stored_s = float(np.median([w for w, _, _ in sto]))
    stored_sweeps_s = float(np.median([s for _, s, _ in sto]))
    cpu = None
    if not args.no_cpu:
        import oracle
        if os.path.exists(oracle.REF_SO):
            ref = oracle.Ref()
            # the reference on the same data and geometry (its bench_compare
            # pipeline; one core, as the reference's solver)
            t0 = time.perf_counter()
            rt = ref.tracer(n, False, (-8, 0, 0), (8, 0, 0), det, 1, spacing, 0.0, views, quarter)
            rt.reconstruct(proj.reshape(views, det).astype(np.float64), beta=beta, tolerance=0, max_sweeps=sweeps)
            ref_polar = time.perf_counter() - t0
            _, ref_otf = ref.cartesian_mart(n, False, (-8, 0, 0), (8, 0, 0), det, 1, spacing, 0.0, views,
                                            proj.astype(np.float64), beta=beta, sweeps=sweeps, stored=False)
            cpu = {"value": ref_otf / ref_polar, "unit": "x", "cores": 1, "kind": "reference",
                   "sample": f"unmodified reference: polar cache build + {sweeps} sweeps {ref_polar:.2f} s, "
                             f"Cartesian Siddon on the fly {ref_otf:.2f} s (acceptance_9 gate >= 1.4, paper 2.5)",
                   "polar_seconds": ref_polar, "cartesian_otf_seconds": ref_otf}
    line = {
        "metric": "USPG vs Cartesian Siddon MART speedup (cmp, acceptance_9 config)",
        "value": otf_sweeps_s / polar_s, "unit": "x", "n_gpus": 1, "steps": reps, "warmup": args.warmup,
        "ms_per_step": polar_s * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic: seeded random-ellipse phantom on square_2d(256), binary projections",
        "config": {"workload": "cmp", "n": n, "detectors": det, "spacing": spacing, "views": views,
                   "sweeps": sweeps, "beta": beta, "l2": "small problem, L2-resident"},
        "speed": {"polar_seconds": polar_s, "polar_sweeps_seconds": polar_sweeps_s,
                  "cartesian_otf_seconds": otf_sweeps_s, "cartesian_stored_seconds": stored_s,
                  "cartesian_stored_sweeps_seconds": stored_sweeps_s,
                  "speedup_vs_otf": otf_sweeps_s / polar_s, "speedup_vs_stored": stored_s / polar_s,
                  "cartesian_levels": otf[0][2]["levels"]},
        "memory": memory, "cpu_baseline": cpu, "e2e": None, "roofline": None,
        "gpu_launches": None,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: the configuration's iteration count for c1-c4 — one whole "
                         "reconstruction, C2: 20 — and 5 for c5, cmp and the reference arm)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--problems", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--length-model", action="store_true",
                    help="also time the length-weighted projector over the stack (not part of the step)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.steps is None:
        args.steps = 5
        if args.impl != "reference" and args.config in ("c1", "c2", "c3", "c4"):
            from paper_2208_12964_b200 import workloads
            args.steps = int(workloads.make(args.config).sweeps)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.config == "c5":
        bench_c5(args, rank, world, local)
        return
    if args.config == "cmp":
        bench_cmp(args, rank, world, local)
        return

    import torch
    import torch.distributed as dist

    import paper_2208_12964_b200 as ub
    from paper_2208_12964_b200 import dist as udist
    from paper_2208_12964_b200 import uscg, workloads

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    wl = workloads.make(args.config, problems=args.problems)
    S = wl.problems
    ctx = ub.Context(local)
    # one stream for torch and the library: events time the launching stream
    # (the legacy default stream's handle is 0, which the ABI reads as "the
    # context's own stream")
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)

    # ---- precompute (geometry only; reported separately like ReconReport::seconds) ----
    t0 = time.perf_counter()
    tracer = ub.Tracer(wl.geom, wl.spec, False, ctx=ctx)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    # weak scaling: every rank reconstructs its own stack of S slices
    wl.seed = udist.rank_seed(wl.seed, rank)
    truth = workloads.phantom_fields(wl, S)
    proj = ub.project_stack(tracer, truth.astype(np.float32))
    proj = workloads.add_noise(wl, proj).astype(np.float32)
    t0 = time.perf_counter()
    levels = tracer.build_schedule()
    t_sched = time.perf_counter() - t0
    info = tracer.info()
    counts = tracer.trace_counts().reshape(-1).astype(np.int64)
    units = counts.size
    nz = proj.reshape(S, -1) != 0
    U = int((nz * counts[None, :]).sum())            # ray-voxel updates per iteration
    Lnz = int(nz.sum())                               # non-skipped (problem, line) pairs
    C = int(info["chords_per_sweep"])                 # chords traced per iteration (shared by the stack)
    B = 8 * U + 20 * C + 8 * units + 4 * Lnz         # algorithmic HBM bytes per iteration

    # ---- device-resident state (interleaved, device-native layout) ----
    Sp = ub.problem_stride(S)
    cells = info["cell_count"]
    pin = np.zeros((units, Sp), np.float32)
    pin[:, :S] = proj.reshape(S, units).T
    proj_d = torch.from_numpy(pin).cuda()
    field_d = torch.ones((cells, Sp), dtype=torch.float32, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    L = ub.load()
    cfg = uscg._Cfg(wl.beta, 0.0, 1, 1.0, 0.0)
    rep = (uscg._Report * S)()
    flags = uscg.DEVICE_POINTERS | uscg.LAYOUT_INTERLEAVED

    def step_dev(sweeps=1):
        cfg.max_sweeps = sweeps
        uscg._check(L.uscg_reconstruct(tracer.h, uscg.C.c_void_p(proj_d.data_ptr()), S, uscg.C.byref(cfg),
                                       uscg.C.c_void_p(field_d.data_ptr()), 1, rep, flags))

    for _ in range(args.warmup):
        step_dev()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    # (1) headline: K iterations as one reconstruct call, run back to back like
    #     any multi-iteration reconstruction (cross-sweep pipelining); the
    #     working set (field + projections + schedule) exceeds L2
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ub.launch_count()
    flush.fill_(1.0)
    torch.cuda.synchronize()
    e0.record(stream)
    step_dev(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    launches = ub.launch_count() - launches0
    t_ms = e0.elapsed_time(e1)
    mart_s = rep[0].seconds
    # (2) isolated iterations: one call per iteration, L2 flushed before each
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    mart_iso = 0.0
    for k in range(args.steps):
        flush.fill_(float(k))
        ev[k][0].record(stream)
        step_dev(1)
        ev[k][1].record(stream)
        mart_iso += rep[0].seconds
    torch.cuda.synchronize()
    clk = clocks.stop()
    t_iso = float(sum(a.elapsed_time(b) for a, b in ev))
    t_ms, mart_s, t_iso, mart_iso = udist.max_over_ranks([t_ms, mart_s, t_iso, mart_iso], device="cuda")
    ms_per_step = t_ms / args.steps
    value = U * world / (ms_per_step * 1e-3)
    isolated = {"ms_per_iteration": t_iso / args.steps, "updates_per_s": U * world / (t_iso / args.steps * 1e-3),
                "l2": "flushed (256 MiB write) before every iteration; one reconstruct call per iteration"}

    # ---- K2 projector over the whole stack (device-resident, one launch) ----
    out_d = torch.empty((units, Sp), dtype=torch.float32, device="cuda")

    def project_dev():
        uscg._check(L.uscg_project(tracer.h, uscg.C.c_void_p(field_d.data_ptr()), S,
                                   uscg.C.c_void_p(out_d.data_ptr()), flags))

    project_dev()
    pe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for k in range(args.steps):
        flush.fill_(float(k))
        pe[k][0].record(stream)
        project_dev()
        pe[k][1].record(stream)
    torch.cuda.synchronize()
    tp = float(sum(a.elapsed_time(b) for a, b in pe)) / args.steps
    U_all = int(counts.sum()) * S
    Bp = 4 * U_all + 20 * C + 8 * units + 4 * units * Sp
    projector = {"ms": tp, "updates_per_s": U_all / (tp * 1e-3), "achieved_gbs": Bp / (tp * 1e-3) / 1e9,
                 "algorithmic_bytes": Bp, "bytes_model": "4*U_all + 20*C + 8*(views*lines) + 4*(views*lines)*S_pad"}
    # length-weighted model (phantom.cpp:213-269) over the whole stack, one
    # call (opt-in: it is not part of the step, and would dominate the
    # command's launch list)
    if args.length_model:
        lw0, lw1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        lw0.record(stream)
        uscg._check(L.uscg_project(tracer.h, uscg.C.c_void_p(field_d.data_ptr()), S,
                                   uscg.C.c_void_p(out_d.data_ptr()), flags | uscg.MODEL_LENGTH))
        lw1.record(stream)
        torch.cuda.synchronize()
        tlw = lw0.elapsed_time(lw1)
        projector["length_weighted"] = {"ms": tlw, "problems": S, "rays_per_s": units * S / (tlw * 1e-3),
                                        "model": "fp64 ray walk per (view, line, 8-problem chunk); cuts at the "
                                                 "radial boundaries inside each chord's sector range"}

    # ---- e2e through the C ABI with pinned host buffers ----
    # K independent stacks (one per step) in one uscg_reconstruct_batch call:
    # every step uploads its projections and initial field and downloads its
    # field inside the timed region; the library overlaps stack k+1's upload
    # and stack k-1's download with stack k's solve (two copy streams).
    e2e = None
    if not args.no_e2e:
        p_host = proj.reshape(S, units)
        stacks = [torch.from_numpy(p_host.copy()).pin_memory() for _ in range(args.steps)]
        # reconstruct (solver.cpp:166-169): the field starts at cfg.f_init, so a
        # step's inputs are its projections and its result the field
        fields = [torch.empty((S, cells), dtype=torch.float32).pin_memory() for _ in range(args.steps)]
        e2e_flags = 0

        def batch_e2e(n):
            pp = (uscg.C.c_void_p * n)(*[uscg.C.c_void_p(x.data_ptr()) for x in stacks[:n]])
            ff = (uscg.C.c_void_p * n)(*[uscg.C.c_void_p(x.data_ptr()) for x in fields[:n]])
            uscg._check(L.uscg_reconstruct_batch(tracer.h, n, pp, S, uscg.C.byref(cfg), ff, 0, None, e2e_flags))

        cfg.max_sweeps = 1
        batch_e2e(min(2, args.steps))  # warm-up (allocations, both staging sets)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        flush.fill_(0.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        batch_e2e(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
        te = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([te], device="cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt[0])
        e2e = {"value": U * world / (te / args.steps * 1e-3), "unit": "updates/s",
               "ms_per_step": te / args.steps,
               "h2d_bytes_per_step": int(stacks[0].numel() * 4),
               "d2h_bytes_per_step": int(fields[0].numel() * 4),
               "api": "uscg_reconstruct_batch over the K steps' stacks (reconstruct: field from cfg.f_init; "
                      "pinned host buffers; each step's upload and download overlapped with the neighbouring "
                      "steps' solves)"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peak, peak_kind = hbm_peak()
    t_mart = mart_s / args.steps  # the MART kernel's device time (CUDA events on its stream) per iteration
    achieved = B / t_mart / 1e9
    traffic = None
    try:
        with open(TRAFFIC_FILE) as f:
            tj = json.load(f)
        if tj.get("config") == args.config:
            traffic = tj.get("dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_kind": peak_kind,
                "kernel": mart_kernel_name(Sp, tracer.info()["executor"]),
                "algorithmic_bytes_per_iteration": B, "dependency_levels_per_iteration": levels,
                "launches": "one persistent launch per reconstruct call (all K iterations); achieved = "
                            "B * K / device time of that launch",
                "avg_time_per_level_us": 1e6 * t_mart / max(levels, 1),
                "bytes_model": "8*U + 20*C + 8*(views*lines) + 4*L_nonzero (DESIGN.md §5)"}

    cpu = None
    if not args.no_cpu and world == 1:
        threads = max(1, os.cpu_count() or 1)
        sample = min(S, 2 * threads)
        v, wall, upd, used = cpu_run(wl, proj, sample, 2, threads)
        cpu = {"value": v, "unit": "updates/s", "cores": used, "kind": "port",
               "sample": f"{sample} of {S} slices x 2 sweeps, one slice per host thread ({wall:.1f} s wall); "
                         f"oracle C restatement (bit-exact to the reference library on its configs)"}
        try:
            ra = ref_lib_analogue(1)
            if ra:
                cpu["reference_lib_analogue"] = ra
        except Exception as e:  # the reference build is optional on the box
            cpu["reference_lib_analogue"] = {"error": str(e)[:200]}

    line = {
        "metric": metric_name(args.config), "value": value, "unit": "updates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: seeded random-ellipse phantoms per slice, binary projections, 1% Gaussian noise",
        "config": config_dict(wl, args),
        "ms_per_iteration": ms_per_step, "updates_per_iteration": U * world, "chords_per_iteration": C,
        "roofline": roofline, "isolated_iteration": isolated, "projector": projector, "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk,
        "precompute": {"generator_s": t_gen, "schedule_s": t_sched, "levels_per_iteration": levels,
                       "records": info["records"], "cache_bytes": info["cache_bytes"],
                       "wave_build_s": tracer.info()["wave_build_s"],
                       "wave_requirements": tracer.info()["wave_requirements"]},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
