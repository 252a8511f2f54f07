#!/usr/bin/env python
"""Benchmark: ms per Sp-MART iteration and ray-voxel updates/s on the USPG
slice stack (BASELINE.json configs[1], "C2"), plus % of the HBM roofline, with
the USCG cone-beam configurations (configs[2], configs[3]: "C3", "C4") measured
in the same run and nested in the line (`uscg`).

A step is one MART iteration (one full sweep over every view and line) of all
S problems of the stack. `value` is measured on device-resident data with
CUDA events; `e2e` runs the same step through the C ABI with pinned host
buffers (projections H2D, field D2H inside the timed region).

    python bench.py [--gpus N --steps K --warmup W --config c2 --impl ours|reference]

Multi-GPU: `--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU). C2 shards the config's 128
slices across the ranks (slices are independent problems, no collective on the
data path; strong scaling); C1/C3/C4 do not shard (the reference's update
within a view is sequential) and run one replica per rank. Timing = max over
ranks of the device time.

`--impl reference` times the reference's CPU path on the box's host cores:
the oracle restatement (oracle/, pinned bit-exactly to the unmodified
reference library) on the same config — the whole 128-slice stack per step,
one slice per host thread — and never loads the product library.
"""
from __future__ import annotations

import argparse
import json
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
PRODUCT_SO = "libuscg_b200.so"


def hbm_peak():
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def product_loaded() -> bool:
    try:
        with open("/proc/self/maps") as f:
            return PRODUCT_SO in f.read()
    except OSError:
        return False


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
        return self

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
# bounded CPU samples per configuration: (problems, views) per step; None = all
CPU_SAMPLE = {"c1": (None, None), "c2": (None, None), "c3": (None, None), "c4": (None, 8)}


class OracleStack:
    """The oracle's reconstruct() over a stack of problems, one problem per
    host thread (reconstruct is single-threaded by design, solver.cpp:76-162;
    slices are independent, SURVEY.md §8(d) CPU protocol). Rays come from the
    oracle's own generators: nothing here loads the product library."""

    def __init__(self, wl, threads: int, views=None):
        import oracle

        self.orc = oracle.Orc()
        self.wl = wl
        self.grid = oracle.OrcGrid.of(wl.spec)
        self.src, self.det = self.orc.rays_for(wl.geom)
        th = wl.geom.thetas()
        self.views = th.size if views is None else min(int(views), th.size)
        self.thetas = th[: self.views]
        self.lines = wl.geom.lines()
        self.threads = max(1, threads)
        self.caches = [self.orc.cache(self.grid, self.src, self.det) for _ in range(self.threads)]

    def _pool(self, n, fn):
        nxt = [0]
        lock = threading.Lock()

        def worker(c):
            while True:
                with lock:
                    i = nxt[0]
                    nxt[0] += 1
                if i >= n:
                    return
                fn(i, c)

        ths = [threading.Thread(target=worker, args=(c,)) for c in self.caches[: min(self.threads, n)]]
        for t in ths:
            t.start()
        for t in ths:
            t.join()

    def project(self, truths):
        """Binary projections (phantom.cpp:182-211) of (S, cells) fields."""
        out = np.zeros((truths.shape[0], self.thetas.size, self.lines))

        def fn(i, c):
            out[i] = c.project(self.thetas, truths[i].astype(np.float32).astype(np.float64))

        self._pool(truths.shape[0], fn)
        return out

    def run(self, projs, sweeps: int):
        """reconstruct() of every problem for `sweeps` sweeps over this
        sample's views; returns (wall seconds, updates)."""
        upd = [0] * len(projs)

        def fn(i, c):
            p = np.asarray(projs[i], np.float64).reshape(-1, self.lines)[: self.views]
            _, rep = c.reconstruct(self.thetas, p, beta=self.wl.beta, tolerance=0, max_sweeps=sweeps)
            upd[i] = rep["updates"]

        t0 = time.perf_counter()
        self._pool(len(projs), fn)
        return time.perf_counter() - t0, int(sum(upd))

    def describe(self, n_problems, sweeps, wall):
        S = self.wl.problems
        what = (f"{n_problems} of {S} slices" if S > 1 else "the volume") + \
               (f", {self.views} of {self.wl.geom.views} views" if self.views < self.wl.geom.views else "")
        return (f"{what} x {sweeps} sweep(s) per step, one problem per host thread ({wall:.2f} s wall); oracle C "
                f"restatement (bit-exact to the reference library on its configs; the reference cannot express "
                f"the verbatim config, SURVEY.md §0.1); CPU: {cpu_model()}, {os.cpu_count()} logical cores")


def ref_lib_analogue():
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
    rt = ref.tracer(512, False, g.source, g.detector_center, g.det_u, 1, g.spacing_u, 0.0, g.views, False, 1)
    rng = np.random.default_rng(1)
    truth = ref.phantom(512, False) * rng.uniform(0.5, 1.0)
    p = rt.project(truth)
    f, rep = rt.reconstruct(p, beta=0.05, tolerance=0, max_sweeps=1)
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


def cpu_inputs(wl, stack: OracleStack, problems: int):
    from paper_2208_12964_b200 import workloads
    truth = workloads.phantom_fields(wl, problems)
    return workloads.add_noise(wl, stack.project(truth).astype(np.float32))


def run_reference(args, rank, world):
    """--impl reference: rank 0 times the CPU path on all host threads, one
    step = one full MART iteration of the config's sample (C2: all 128
    slices, measured, not extrapolated)."""
    from paper_2208_12964_b200 import workloads

    if rank != 0:
        return
    wl = workloads.make(args.config, problems=args.problems)
    threads = max(1, os.cpu_count() or 1)
    n_prob, n_views = CPU_SAMPLE.get(args.config, (None, None))
    S = wl.problems if n_prob is None else min(n_prob, wl.problems)
    stack = OracleStack(wl, threads, n_views)
    proj = cpu_inputs(wl, stack, S)
    for _ in range(args.warmup):
        stack.run(proj, 1)
    walls, upds = [], []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        w, u = stack.run(proj, 1)
        walls.append(w)
        upds.append(u)
    total = time.perf_counter() - t0
    value = float(sum(upds)) / float(sum(walls))
    if product_loaded():
        raise RuntimeError("the reference arm mapped the product library")
    line = {
        "impl": "reference", "metric": metric_name(args.config), "value": value, "unit": "updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded random-ellipse phantoms, binary projections, configured noise",
        "config": config_dict(wl, args, world),
        "cpu_baseline": {"value": value, "unit": "updates/s", "cores": min(threads, S), "kind": "port",
                         "cpu": cpu_model(), "sample": stack.describe(S, 1, float(np.mean(walls)))},
        "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "native_product_loaded": False,
    }
    print(json.dumps(line), flush=True)


def metric_name(config):
    return f"ray-voxel updates/s per Sp-MART iteration ({config})"


def config_dict(wl, args, world):
    spec, geom = wl.spec, wl.geom
    stack = wl.problems > 1
    return {"workload": wl.name, "problems": wl.problems, "rings": spec.rings(),
            "sector_law": "reference 4(2k-1)" if spec.ring_counts is None else "round(2*pi*(i+0.5))",
            "cells_per_slice": spec.cells_per_slice(), "slices": spec.slices(), "views": geom.views,
            "detectors": [geom.det_u, geom.det_v], "detector": geom.detector.name.lower(), "beta": wl.beta,
            "iterations_per_reconstruction": wl.sweeps,
            "l2": "timed iterations run back to back in one reconstruct call; working set > L2 "
                  "(field + projections + schedule); 'isolated' repeats with L2 flushed per iteration",
            "parallelism": (f"{wl.problems} slices sharded over {world} GPU(s) (strong scaling)" if stack
                            else f"one replica per GPU ({world})")}


# ---------------------------------------------------------------------------
# GPU arm: MART configurations (C1-C4)
# ---------------------------------------------------------------------------
class Gpu:
    def __init__(self, local):
        import torch

        import paper_2208_12964_b200 as ub
        self.torch, self.ub = torch, ub
        self.local = local
        self.ctx = ub.Context(local)
        # one stream for torch and the library: events time the launching
        # stream (the legacy default stream's handle is 0, which the ABI reads
        # as "the context's own stream")
        self.stream = torch.cuda.Stream(device=local)
        torch.cuda.set_stream(self.stream)
        self.ctx.set_stream(self.stream.cuda_stream)
        self.flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def event(self):
        return self.torch.cuda.Event(enable_timing=True)


def mart_kernel_name(info, P):
    ex = info["executor"]
    if ex == 3:
        cl = int(info.get("wave_ctas", 1) or 1)
        if cl > 1:
            return (f"mart_wave_pair_kernel<{P}, 1, {cl}> (one persistent launch per reconstruct call; task = "
                    f"(view, {P}-problem chunk) on a {cl}-CTA cluster)")
        return f"mart_wave_kernel<{P}> (one persistent launch per reconstruct call; task = (view, {P}-problem chunk))"
    if ex == 4:
        return "mart_tile_kernel (one CTA, the field in shared memory)"
    if ex == 5:
        return ("mart_level_kernel<256, 3> (one launch per dependency level, chained by programmatic dependent "
                "launch; a 256-thread block per line with a non-zero measurement)")
    return (f"mart_flow_kernel<{P}> (one dataflow launch per reconstruct call"
            + ("; task = one line, fed by its precomputed traced list)" if info.get("executor_bytes") else ")"))


def chunk_width(Sp):
    """The library's MART chunk width for a stack of stride Sp (kernels.cu
    chunk_width: a limit of 16 up to 64 problems, else 32)."""
    p = 1
    lim = int(os.environ.get("USCG_CHUNK_WIDTH", 32 if Sp > 64 else 16))
    while p * 2 <= lim and Sp % (p * 2) == 0:
        p *= 2
    return p


def bench_mart(gpu: Gpu, config, args, rank, world, steps=None, warmup=None, cpu=True, e2e=True, iso=True,
               weak=False):
    """One MART configuration: returns the JSON line (rank 0) or None.
    weak: every rank reconstructs a whole stack of its own (distinct seeds)
    instead of its shard of the config's stack."""
    import torch

    from paper_2208_12964_b200 import dist as udist
    from paper_2208_12964_b200 import uscg, workloads

    ub = gpu.ub
    stream = gpu.stream
    steps = args.steps if steps is None else steps
    warmup = args.warmup if warmup is None else warmup
    wl = workloads.make(config, problems=args.problems if config == args.config else None)
    S_all = wl.problems
    stacked = S_all > 1
    lo, hi = udist.shard(S_all, rank, world) if stacked and not weak else (0, S_all)
    if weak:
        wl.seed = udist.rank_seed(wl.seed, rank)
    S = hi - lo

    # ---- precompute (geometry only; reported separately like ReconReport::seconds) ----
    t0 = time.perf_counter()
    tracer = ub.Tracer(wl.geom, wl.spec, False, ctx=gpu.ctx)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    truth = workloads.phantom_fields(wl, S, first=lo)
    proj = workloads.add_noise(wl, ub.project_stack(tracer, truth.astype(np.float32)), first=lo).astype(np.float32)
    del truth
    t0 = time.perf_counter()
    levels = tracer.build_schedule()
    t_sched = time.perf_counter() - t0
    info = tracer.info()
    counts = tracer.trace_counts().reshape(-1).astype(np.int64)
    units = counts.size
    nz = proj.reshape(S, -1) != 0
    U = int((nz * counts[None, :]).sum())             # ray-voxel updates per iteration (this rank)
    Lnz = int(nz.sum())                               # non-skipped (problem, line) pairs
    C = int(info["chords_per_sweep"])                 # chords traced per iteration (shared by the stack)
    E = int(counts.sum())                             # cell visits per iteration of one problem

    # ---- device-resident state (interleaved, device-native layout) ----
    Sp = ub.problem_stride(S)
    P = chunk_width(Sp)
    cells = info["cell_count"]
    pin = np.zeros((units, Sp), np.float32)
    pin[:, :S] = proj.reshape(S, units).T
    proj_d = torch.from_numpy(pin).cuda()
    del pin
    field_d = torch.ones((cells, Sp), dtype=torch.float32, device="cuda")
    L = ub.load()
    cfg = uscg._Cfg(wl.beta, 0.0, 1, 1.0, 0.0)
    rep = (uscg._Report * S)()
    flags = uscg.DEVICE_POINTERS | uscg.LAYOUT_INTERLEAVED

    def step_dev(sweeps=1):
        cfg.max_sweeps = sweeps
        uscg._check(L.uscg_reconstruct(tracer.h, uscg.C.c_void_p(proj_d.data_ptr()), S, uscg.C.byref(cfg),
                                       uscg.C.c_void_p(field_d.data_ptr()), 1, rep, flags))

    for _ in range(warmup):
        step_dev()
    torch.cuda.synchronize()
    info = tracer.info()
    if info["executor"] == 5:
        levels = int(info["levels"])  # the level executor's line levels (the run levels above are the flow executor's)
    if world > 1 and torch.distributed.is_initialized():
        torch.distributed.barrier()
    clocks = Clocks(gpu.local).start()
    # (1) headline: K iterations as one reconstruct call, run back to back like
    #     any multi-iteration reconstruction (cross-sweep pipelining); the
    #     working set (field + projections + schedule) exceeds L2
    e0, e1 = gpu.event(), gpu.event()
    launches0 = ub.launch_count()
    gpu.flush.fill_(1.0)
    torch.cuda.synchronize()
    e0.record(stream)
    step_dev(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    launches = ub.launch_count() - launches0
    t_ms = e0.elapsed_time(e1)
    mart_s = rep[0].seconds
    # (2) isolated iterations: one call per iteration, L2 flushed before each
    t_iso = 0.0
    if iso:
        ev = [(gpu.event(), gpu.event()) for _ in range(steps)]
        for k in range(steps):
            gpu.flush.fill_(float(k))
            ev[k][0].record(stream)
            step_dev(1)
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        t_iso = float(sum(a.elapsed_time(b) for a, b in ev))
    clk = clocks.stop()
    (U_all,) = udist.sum_over_ranks([U], device="cuda") if stacked else (U * world,)
    t_ms, mart_s, t_iso = udist.max_over_ranks([t_ms, mart_s, t_iso], device="cuda")
    ms_per_step = t_ms / steps
    value = U_all / (ms_per_step * 1e-3)

    # ---- K2 projector over the stack (device-resident, one launch); one
    #      problem on N ranks: each rank projects its block of views
    #      (dist.view_subset_tracer over the same record store) ----
    ptr, p_units = tracer, units
    if not stacked and world > 1:
        v0, v1 = udist.shard(info["views"], rank, world)
        ptr = udist.view_subset_tracer(tracer, v0, v1)
        p_units = (v1 - v0) * info["lines"]
    out_d = torch.empty((max(p_units, 1), Sp), dtype=torch.float32, device="cuda")

    def project_dev():
        uscg._check(L.uscg_project(ptr.h, uscg.C.c_void_p(field_d.data_ptr()), S,
                                   uscg.C.c_void_p(out_d.data_ptr()), flags))

    project_dev()
    pe = [(gpu.event(), gpu.event()) for _ in range(max(1, min(steps, 5)))]
    for a, b in pe:
        gpu.flush.fill_(0.5)
        a.record(stream)
        project_dev()
        b.record(stream)
    torch.cuda.synchronize()
    tp = float(sum(a.elapsed_time(b) for a, b in pe)) / len(pe)
    (tp,) = udist.max_over_ranks([tp], device="cuda")
    if ptr is not tracer:
        ptr.close()
    # the whole job over all ranks (stacks: every rank's slices; one problem:
    # every rank's views); frac is per GPU
    S_job = S_all if stacked else 1
    reps = world if stacked else 1
    listed = Sp == 1 and int(info.get("executor_bytes", 0)) > 0
    if listed:  # one problem with the solver's traced lists: project_lists_kernel
        Bp = 8 * E + 12 * units
        p_model = "8*E (u32 list entry + fp32 field gather per cell) + 12*(views*lines) (u64 offsets, output)"
    else:
        Bp = 4 * E * S_job + reps * (20 * C + 8 * units + 4 * units * Sp)
        p_model = ("4*E*S (field gathers) + 20*C (records) + 8*(views*lines) (offsets, measurement index) + "
                   "4*(views*lines)*S_pad (projections written)")
    peak, peak_kind = hbm_peak()
    projector = {"ms": tp, "updates_per_s": E * S_job / (tp * 1e-3), "achieved_gbs": Bp / (tp * 1e-3) / 1e9,
                 "frac": Bp / (tp * 1e-3) / 1e9 / peak / world, "algorithmic_bytes": Bp,
                 "kernel": ("project_stack_kernel" if Sp > 1 else
                            "project_lists_kernel" if listed else "project_kernel<1>"),
                 "parallelism": ("slices sharded" if stacked else
                                 f"views sharded over {world} GPU(s) (dist.view_subset_tracer)" if world > 1
                                 else "one GPU"),
                 "bytes_model": p_model}
    if projector["frac"] > 1:
        projector["note"] = ("above 1: the algorithmic bytes are compared with the HBM copy bandwidth, and part of "
                             "the field gathers are served by L2 (ncu DRAM throughput ~60% of peak for this kernel)")
    del out_d

    # ---- e2e through the C ABI with pinned host buffers ----
    e2e_line = None
    if e2e:
        p_host = proj.reshape(S, units)
        if stacked:
            # K independent stacks (one per step) in one uscg_reconstruct_batch
            # call: every step uploads its projections and downloads its field
            # inside the timed region; the library overlaps stack k+1's upload
            # and stack k-1's download with stack k's solve (two copy streams)
            stacks = [torch.from_numpy(p_host.copy()).pin_memory() for _ in range(steps)]
            fields = [torch.empty((S, cells), dtype=torch.float32).pin_memory() for _ in range(steps)]

            def run_e2e(n):
                pp = (uscg.C.c_void_p * n)(*[uscg.C.c_void_p(x.data_ptr()) for x in stacks[:n]])
                ff = (uscg.C.c_void_p * n)(*[uscg.C.c_void_p(x.data_ptr()) for x in fields[:n]])
                uscg._check(L.uscg_reconstruct_batch(tracer.h, n, pp, S, uscg.C.byref(cfg), ff, 0, None, 0))

            api = ("uscg_reconstruct_batch over the K steps' stacks (reconstruct: field from cfg.f_init; pinned "
                   "host buffers; each step's upload and download overlapped with the neighbouring steps' solves)")
            cfg.max_sweeps = 1
            run_e2e(min(2, steps))  # warm-up (allocations, both staging sets)
            nrun = steps
        else:
            # one reconstruct() call of K iterations from pinned host buffers:
            # projections up, field down, inside the timed region
            stacks = [torch.from_numpy(p_host.copy()).pin_memory()]
            fields = [torch.empty((S, cells), dtype=torch.float32).pin_memory()]
            rep1 = (uscg._Report * S)()

            def run_e2e(n):
                cfg.max_sweeps = n
                uscg._check(L.uscg_reconstruct(tracer.h, uscg.C.c_void_p(stacks[0].data_ptr()), S,
                                               uscg.C.byref(cfg), uscg.C.c_void_p(fields[0].data_ptr()), 0, rep1, 0))

            api = ("uscg_reconstruct of K iterations from pinned host buffers (reconstruct: field from cfg.f_init; "
                   "projections H2D and the field D2H inside the timed region)")
            for _ in range(max(1, min(args.warmup, 3))):
                run_e2e(1)  # warm-up calls on the same buffers (the level executor keeps its launch graph from the second)
            nrun = steps
        torch.cuda.synchronize()
        if world > 1 and torch.distributed.is_initialized():
            torch.distributed.barrier()
        a, b = gpu.event(), gpu.event()
        torch.cuda.synchronize()
        a.record(stream)
        run_e2e(nrun)
        b.record(stream)
        torch.cuda.synchronize()
        (te,) = udist.max_over_ranks([a.elapsed_time(b)], device="cuda")
        h2d = int(stacks[0].numel() * 4)
        d2h = int(fields[0].numel() * 4)
        e2e_line = {"value": U_all / (te / steps * 1e-3), "unit": "updates/s", "ms_per_step": te / steps,
                    "h2d_bytes_per_step": h2d if stacked else h2d // steps,
                    "d2h_bytes_per_step": d2h if stacked else d2h // steps, "api": api}
        del stacks, fields

    if rank != 0:
        tracer.close()
        return None

    t_mart = mart_s / steps  # the MART kernel's device time (CUDA events on its stream) per iteration
    exe_bytes = int(info.get("executor_bytes", 0))
    if info["executor"] == 3:
        chunks = Sp // P
        B = 8 * U + 8 * E * chunks + 4 * units * Sp + 8 * units * chunks
        model = ("8*U (fp32 field read+write of every update) + 8*E*chunks (the wave's traced lists: one uint2 per "
                 "cell visit per P-problem chunk) + 4*(views*lines)*S_pad (measurements) + 8*(views*lines)*chunks "
                 "(list offsets, requirements)")
    elif exe_bytes:
        B = 12 * U + 4 * Lnz + 16 * units
        model = ("12*U (u32 traced-list entry + fp32 field read+write per update) + 4*L_nonzero (measurement) + "
                 "16*(views*lines) (u64 list offset, schedule order/successor metadata)")
    else:
        B = 8 * U + 20 * C + 8 * units + 4 * Lnz
        model = "8*U + 20*C (records, traced every sweep) + 8*(views*lines) + 4*L_nonzero"
    achieved = B / t_mart / 1e9
    traffic = None
    try:
        with open(TRAFFIC_FILE) as f:
            tj = json.load(f)
        if config in tj:
            traffic = tj[config].get("dram_bytes_per_iteration")
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_unit": "DRAM bytes per iteration (ncu, profiles/)",
                "peak_kind": peak_kind, "kernel": mart_kernel_name(info, P),
                "algorithmic_bytes_per_iteration": B, "bytes_model": model,
                "levels_per_iteration": levels,
                "launches": ("one launch per dependency level and iteration; achieved = B * K / device time of the "
                             "reconstruct call's launches" if info["executor"] == 5 else
                             "one persistent launch per reconstruct call (all K iterations); achieved = "
                             "B * K / device time of that launch")}
    # what binds each executor, measured
    notes = {
        "c2": ("the per-line chain and the SMs' scattered 128-byte row traffic, mostly served by L2 "
               "(profiles/r2_row_microbench.md): the fraction compares the algorithmic bytes with HBM"),
        "c3": ("latency: the dependency chain's 1269 line levels at ~3.4 us each (one gather round trip, a two-warp "
               "sum, the factor, the stores and the hand-over to the next level's waiting grid); its 26 MB field "
               "stays in L2"),
        "c4": ("scattered 4-byte read-modify-writes on a 211 MB field: ~90 G updates/s, the rate a microbenchmark "
               "of that access pattern reaches (profiles/r2_sector_microbench.md)"),
        "c1": "latency: one CTA, one block barrier per dependency level",
    }
    if config in notes:
        roofline["bound_detail"] = notes[config]

    cpu_line = None
    if cpu and world == 1 and not args.no_cpu:
        threads = max(1, os.cpu_count() or 1)
        n_prob, n_views = CPU_SAMPLE.get(config, (None, None))
        ns = S if n_prob is None else min(S, n_prob)
        stk = OracleStack(wl, threads, n_views)
        wall, upd = stk.run(proj[:ns], 1)
        cpu_line = {"value": upd / wall, "unit": "updates/s", "cores": min(threads, ns), "kind": "port",
                    "cpu": cpu_model(), "sample": stk.describe(ns, 1, wall)}
        del stk

    line = {
        "metric": metric_name(config), "value": value, "unit": "updates/s", "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if stacked else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: seeded random phantoms (per slice), binary projections, configured noise",
        "config": config_dict(wl, args, world),
        "ms_per_iteration": ms_per_step, "updates_per_iteration": U_all, "chords_per_iteration": C,
        "roofline": roofline, "projector": projector, "cpu_baseline": cpu_line, "e2e": e2e_line,
        "gpu_launches": int(launches), "clocks": clk,
        "device_bytes": {"record_store": int(info["cache_bytes"]), "executor_lists": exe_bytes,
                         "note": "executor_lists = the p-fold-expanded traced lists / schedule the MART executor "
                                 "reads instead of rotating the record store every sweep"},
        "precompute": {"generator_s": t_gen, "schedule_s": t_sched, "levels_per_iteration": levels,
                       "records": info["records"], "wave_build_s": info["wave_build_s"],
                       "wave_requirements": info["wave_requirements"]},
    }
    if iso:
        line["isolated_iteration"] = {"ms_per_iteration": t_iso / steps, "updates_per_s": U_all / (t_iso / steps * 1e-3),
                                      "l2": "flushed (256 MiB write) before every iteration; one reconstruct call "
                                            "per iteration"}
    if stacked:
        line["per_gpu_slices"] = S
    tracer.close()
    return line


def bench_store_fed(gpu: Gpu, config, args, sweeps=3):
    """The same configuration with the MART executor fed by the
    symmetry-compressed record store (every line rotated and expanded from
    the one-view store each sweep; no p-fold-expanded lists)."""
    prev = {k: os.environ.get(k) for k in ("USCG_MART_MODE", "USCG_FLOW_LISTS")}
    os.environ["USCG_MART_MODE"] = "flow"
    os.environ["USCG_FLOW_LISTS"] = "0"
    try:
        ln = bench_mart(gpu, config, args, 0, 1, steps=sweeps, warmup=1, cpu=False, e2e=False, iso=False)
    finally:
        for k, v in prev.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return {"ms_per_iteration": ln["ms_per_iteration"], "updates_per_s": ln["value"],
            "kernel": ln["roofline"]["kernel"], "executor_lists_bytes": ln["device_bytes"]["executor_lists"],
            "record_store_bytes": ln["device_bytes"]["record_store"], "iterations": sweeps,
            "roofline_frac": ln["roofline"]["frac"], "bytes_model": ln["roofline"]["bytes_model"]}


# ---------------------------------------------------------------------------
# C5: coefficient generation, rotated reuse, USPG -> CG resampling
# ---------------------------------------------------------------------------
def bench_c5(args, rank, world, local):
    """BASELINE configs[4]. Three device-timed legs:
    (1) the first-view generator over the 1024x1024 panel (rays/s; device time
    reported by the library, count + scan + write + annotate); (2) rotated
    reuse: every (view, line) of 180 views served from the one-view record
    store, |active| + index checksum per line (lines/s); (3) resampling a
    seeded U[0,1] 512-ring x 512-slice USPG volume to 1024 x 1024 x 512 (8 B
    per output pixel). N > 1 ranks split detector rows, views and slices
    (strong scaling); the generator's one exchange assembles the full record
    store on every rank (dist.assemble_cache)."""
    import torch
    import torch.distributed as dist

    import paper_2208_12964_b200 as ub
    from paper_2208_12964_b200 import dist as udist
    from paper_2208_12964_b200 import uscg, workloads

    gpu = Gpu(local)
    ctx, stream = gpu.ctx, gpu.stream
    wl = workloads.make("c5")
    spec, geom = wl.spec, wl.geom
    L = ub.load()
    src, det = geom.first_view_rays()
    lines = geom.lines()
    rows = geom.det_v
    r0, r1 = udist.shard(rows, rank, world)
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

    exchange_ms = 0.0
    if world > 1:
        local_tr = ub.Tracer.from_rays(spec, src[mine], det[mine], 1, ctx=ctx)
        part = local_tr.copy_cache(device=True)
        local_tr.close()
        torch.cuda.synchronize()
        dist.barrier()
        x0, x1 = gpu.event(), gpu.event()
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
    v0, v1 = udist.shard(geom.views, rank, world)
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
    clocks = Clocks(local).start()
    e0, e1 = gpu.event(), gpu.event()
    launches0 = ub.launch_count()
    e0.record(stream)
    for _ in range(args.steps):
        reuse()
    e1.record(stream)
    torch.cuda.synchronize()
    reuse_ms = e0.elapsed_time(e1) / args.steps
    chords = inf["records"] * nv
    cnt_ref = tr.trace_counts()[v0:v1].reshape(-1)
    reuse_ok = bool(np.array_equal(counts_d.cpu().numpy().astype(np.uint32), cnt_ref))
    tr.close()

    # (3) resample this rank's slices of a seeded U[0,1] volume
    sl0, sl1 = udist.shard(spec.slices(), rank, world)
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
    #     perturbed copy (mae / rmse / ssim per slice, ssim_volume's shared range)
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
    rays_all, recs_all, px_all = udist.sum_over_ranks([rays_mine, recs, px], device="cuda")

    if rank != 0:
        return
    peak, peak_kind = hbm_peak()
    gen_bytes = 20 * recs_all + 4 * (lines + 1)
    res_bytes = 8 * px_all

    def roof(bytes_, ms, kernel, model, bound="hbm"):
        a = bytes_ / (ms * 1e-3) / 1e9
        return {"bound": bound, "achieved": a, "peak": peak, "unit": "GB/s", "frac": a / peak, "traffic": None,
                "peak_kind": peak_kind, "kernel": kernel, "bytes_model": model}

    cpu = None
    if not args.no_cpu and world == 1:
        import oracle

        orc = oracle.Orc()
        og = oracle.OrcGrid.of(spec)
        osrc, odet = orc.rays_for(geom)
        pick = np.random.default_rng(5).choice(lines, 512, replace=False)
        t0 = time.perf_counter()
        oc = orc.cache(og, osrc[pick], odet[pick])
        wall = time.perf_counter() - t0
        cpu = {"value": pick.size / wall, "unit": "rays/s", "cores": 1, "kind": "port", "cpu": cpu_model(),
               "sample": f"oracle C restatement of precompute_first_view on {pick.size} random rays of the panel "
                         f"({wall:.1f} s, {int(oc.offsets[-1])} records)"}
    value = rays_all / ((g_ms + exchange_ms) * 1e-3)
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
        "roofline": roof(gen_bytes, g_ms, "generate_bound_kernel + generate_slot_kernel + compact_records_kernel + "
                         "annotate_kernel", "20*records + 4*(lines+1) written (SURVEY.md §8(d)); fp64-compute "
                         "bound, see DESIGN.md §4.2"),
        "generator": {"ms": g_ms, "exchange_ms": exchange_ms, "rays": rays_all, "records": recs_all,
                      "records_per_s": recs_all / ((g_ms + exchange_ms) * 1e-3)},
        "rotated_reuse": {"ms": reuse_ms, "views": geom.views, "lines_per_s": world * nv * lines / (reuse_ms * 1e-3),
                          "chords_per_s": world * chords / (reuse_ms * 1e-3), "counts_match_library": reuse_ok,
                          "bound": "fp64 rotation + L1-served record reuse (each record read once per line, "
                                   "all views served from L1): not an HBM figure",
                          "hbm_bytes_model": "20*records + 12*views*lines (records once, counts + checksums out)"},
        "resample": {"ms": res_ms, "pixels": px_all, "pixels_per_s": px_all / (res_ms * 1e-3),
                     "roofline": roof(res_bytes, res_ms, "tiled_resample_kernel (per 32x32 tile: coalesced cell runs staged in shared memory)",
                                      "8 B per output pixel (SURVEY.md §8(d))")},
        "metrics": {"ms": met_ms, "slices": spec.slices(), "ssim_volume": float(m_ssim.mean()),
                    "rmse_volume": float(m_rmse.mean()), "pixels_per_s": px_all / (met_ms * 1e-3),
                    "bound": "fp64 window arithmetic (SSIM), not HBM"},
        "cpu_baseline": cpu, "e2e": None, "gpu_launches": int(launches), "clocks": clk,
    }
    print(json.dumps(line), flush=True)


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
    from paper_2208_12964_b200 import workloads

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
            t0 = time.perf_counter()
            rt = ref.tracer(n, False, (-8, 0, 0), (8, 0, 0), det, 1, spacing, 0.0, views, quarter)
            rt.reconstruct(proj.reshape(views, det).astype(np.float64), beta=beta, tolerance=0, max_sweeps=sweeps)
            ref_polar = time.perf_counter() - t0
            _, ref_otf = ref.cartesian_mart(n, False, (-8, 0, 0), (8, 0, 0), det, 1, spacing, 0.0, views,
                                            proj.astype(np.float64), beta=beta, sweeps=sweeps, stored=False)
            cpu = {"value": ref_otf / ref_polar, "unit": "x", "cores": 1, "kind": "reference", "cpu": cpu_model(),
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
# length-weighted MART on the polar grid's (voxel, chord length) lists
# ---------------------------------------------------------------------------
def bench_lw(args, rank, world, local):
    """uscg_tracer_length_system on C1 and C3: the (voxel index, chord length)
    lists of the LengthWeighted model (phantom.cpp:213-269) built on the device,
    then K iterations of the reference's weighted row action (siddon.cpp:141-154)
    on the USPG / USCG field, one launch per dependency level. Beside it: the
    binary-model executor on the same geometry, and the oracle's weighted MART
    on the same lists on one host core. Rank 0 only (one problem)."""
    import torch

    import paper_2208_12964_b200 as ub
    from paper_2208_12964_b200 import workloads

    if rank != 0:
        return
    torch.cuda.set_device(local)
    peak, peak_kind = hbm_peak()
    out = {}
    clocks = Clocks(local).start()
    launches0 = ub.launch_count()
    for name in ("c1", "c3"):
        wl = workloads.make(name)
        spec, geom = wl.spec, wl.geom
        tr = ub.Tracer(geom, spec, False)
        truth = workloads.phantom_fields(wl, 1)[0].astype(np.float32)
        proj = ub.project_stack(tr, truth[None], model="length")[0].reshape(-1)
        t0 = time.perf_counter()
        ls = ub.LengthSystem(tr)
        build_s = time.perf_counter() - t0
        inf = ls.info()
        K = int(wl.sweeps)
        cfg = ub.SolverConfig(beta=wl.beta, tolerance=0, max_sweeps=K)
        for _ in range(max(1, min(args.warmup, 2))):
            ls.reconstruct(proj, cfg)
        field, sec = ls.reconstruct(proj, cfg)
        ms_it = 1e3 * sec / K
        bres = ub.reconstruct(ub.ProjectionSet(geom, ub.project_stack(tr, truth[None])[0].astype(np.float64)), spec,
                              cfg, tr)
        cpu = None
        exp = ls.export()
        live = np.diff(exp[0].astype(np.int64))[proj > 0]  # zero measurements are skipped (siddon.cpp:143)
        U = int(live.sum())
        if not args.no_cpu:
            import oracle
            orc = oracle.Orc()
            off, idx, w = exp
            t0 = time.perf_counter()
            orc.weighted_mart(off, idx, w.astype(np.float64), proj.astype(np.float64), beta=wl.beta, sweeps=1,
                              cells=spec.cell_count())
            cw = time.perf_counter() - t0
            cpu = {"value": U / cw, "unit": "updates/s", "cores": 1, "kind": "port", "cpu": cpu_model(),
                   "sample": f"oracle weighted_update restatement, one sweep over the same lists ({cw:.2f} s)"}
        re = None
        if name == "c1":  # closure: length-weighted projections of the result against the data
            off, idx, w = exp
            rows = geom.views * geom.lines()
            re = np.bincount(np.repeat(np.arange(rows), np.diff(off.astype(np.int64))),
                             weights=w.astype(np.float64) * field[idx], minlength=rows)
        B = 20 * U + 8 * proj.size  # u32 index + f32 length + field read (sum), read + write (update)
        out[name] = {
            "ms_per_iteration": ms_it, "updates_per_iteration": U,
            "updates_per_s": U / (ms_it * 1e-3), "iterations": K, "levels": inf["levels"],
            "lists": {"entries": inf["entries"], "device_bytes": inf["device_bytes"],
                      "device_build_ms": inf["precompute_ms"], "build_with_host_schedule_s": build_s},
            "roofline": {"bound": "hbm", "achieved": B / (ms_it * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": B / (ms_it * 1e-3) / 1e9 / peak, "traffic": None, "peak_kind": peak_kind,
                         "kernel": "csr_level_kernel (one launch per dependency level, a block per line)",
                         "bytes_model": "20 B per list entry of a line with a non-zero measurement (u32 index, "
                                        "f32 length, field read for the sum, read + write for the update) + 8 B "
                                        "per line (offset, measurement)"},
            "binary_model_ms_per_iteration": 1e3 * bres.report.seconds / K,
            "closure_mean_abs_residual": None if re is None else float(np.abs(re - proj)[proj > 0].mean()),
            "cpu_baseline": cpu,
        }
        ls.close()
        tr.close()
    clk = clocks.stop()
    c3 = out["c3"]
    line = {
        "metric": "length-weighted MART updates/s on USCG (c3, (voxel, chord length) lists)",
        "value": c3["updates_per_s"], "unit": "updates/s", "n_gpus": 1, "steps": c3["iterations"],
        "warmup": args.warmup, "ms_per_step": c3["ms_per_iteration"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: seeded phantoms, length-weighted projections of the same model",
        "config": {"workload": "lw", "parts": ["c1", "c3"], "l2": "C3: lists of ~1 GB exceed L2; C1 is L2-resident"},
        "roofline": c3["roofline"], "cpu_baseline": c3["cpu_baseline"], "e2e": None,
        "gpu_launches": int(ub.launch_count() - launches0), "clocks": clk, "c1": out["c1"], "c3": out["c3"],
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# entry
# ---------------------------------------------------------------------------
def relaunch(n):
    """`--gpus N` outside torchrun: re-exec under torch.distributed.run with
    N ranks on this node (rendezvous on 127.0.0.1)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


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
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline legs")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-uscg", action="store_true", help="C2 line without the nested C3/C4 measurements")
    ap.add_argument("--no-store-fed", action="store_true", help="skip the store-fed (no lists) executor timing")
    ap.add_argument("--no-weak", action="store_true", help="N > 1: skip the weak-scaling extra key")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch(args.gpus)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; reporting n_gpus={world}", file=sys.stderr)

    if args.steps is None:
        args.steps = 5
        if args.impl != "reference" and args.config in ("c1", "c2", "c3", "c4"):
            from paper_2208_12964_b200 import workloads
            args.steps = int(workloads.make(args.config).sweeps)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        if args.config == "c5":
            bench_c5(args, rank, world, local)
        elif args.config == "cmp":
            bench_cmp(args, rank, world, local)
        elif args.config == "lw":
            bench_lw(args, rank, world, local)
        else:
            gpu = Gpu(local)
            line = bench_mart(gpu, args.config, args, rank, world)
            if world > 1 and args.config == "c2" and not args.no_weak:
                # extra key: weak scaling, one whole 128-slice stack per GPU
                # (the headline `value` shards the config's stack)
                wk = bench_mart(gpu, "c2", args, rank, world, cpu=False, e2e=False, iso=False, weak=True)
                if rank == 0:
                    line["weak_scaling"] = {"value": wk["value"], "unit": "updates/s",
                                            "ms_per_step": wk["ms_per_step"],
                                            "slices_per_gpu": wk["per_gpu_slices"],
                                            "note": "every GPU reconstructs its own 128-slice stack (distinct seeds); "
                                                    "value = all GPUs' updates / the slowest GPU's time"}
            if rank == 0 and args.config == "c2" and world == 1 and not args.no_store_fed:
                line["store_fed"] = bench_store_fed(gpu, "c2", args)
            if rank == 0 and args.config == "c2" and world == 1 and not args.no_uscg:
                # the metric is "... on USCG": the cone-beam configurations,
                # one replica, each a whole reconstruction's iterations
                uscg_legs = {}
                for c in ("c3", "c4"):
                    sub = bench_mart(gpu, c, args, 0, 1, steps=_sweeps(c), warmup=2,
                                     iso=False)
                    uscg_legs[c] = {k: sub[k] for k in ("metric", "value", "unit", "ms_per_iteration", "steps",
                                                        "warmup", "updates_per_iteration", "roofline", "projector",
                                                        "cpu_baseline", "e2e", "gpu_launches", "clocks",
                                                        "device_bytes", "precompute", "config")}
                line["uscg"] = uscg_legs
            if rank == 0:
                print(json.dumps(line), flush=True)
    finally:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()


def _sweeps(config):
    from paper_2208_12964_b200 import workloads
    return int(workloads.make(config).sweeps)


if __name__ == "__main__":
    main()
