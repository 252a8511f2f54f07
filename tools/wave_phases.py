"""Per-task phase times of the wave MART executor (diagnostics, never a bench
number): python tools/wave_phases.py [config] [sweeps] -> one reconstruct call
with USCG_SWEEP_PROFILE stamps, then per line the mean time waiting for the
line's other-view requirements, gathering, reducing (factor) and storing, and
the mean number of tasks in flight."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path = os.path.join(tempfile.mkdtemp(), "prof.bin")
os.environ["USCG_SWEEP_PROFILE"] = path
os.environ.setdefault("USCG_MART_MODE", "wave")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2208_12964_b200 as ub  # noqa: E402
from paper_2208_12964_b200 import uscg, workloads  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
wl = workloads.make(cfgname)
S = wl.problems
tracer = ub.Tracer(wl.geom, wl.spec, False)
truth = workloads.phantom_fields(wl, S).astype(np.float32)
proj = ub.project_stack(tracer, truth)
info = tracer.info()
units = info["views"] * info["lines"]
Sp = ub.problem_stride(S)
pin = np.zeros((units, Sp), np.float32)
pin[:, :S] = proj.reshape(S, units).T
proj_d = torch.from_numpy(pin).cuda()
field_d = torch.ones((info["cell_count"], Sp), dtype=torch.float32, device="cuda")
L = ub.load()
flags = uscg.DEVICE_POINTERS | uscg.LAYOUT_INTERLEAVED
rep = (uscg._Report * S)()
for k in range(2):  # warm-up call builds the lists, then the profiled call
    cfg = uscg._Cfg(wl.beta, 0.0, sweeps, 1.0, 0.0)
    uscg._check(L.uscg_reconstruct(tracer.h, uscg.C.c_void_p(proj_d.data_ptr()), S, uscg.C.byref(cfg),
                                   uscg.C.c_void_p(field_d.data_ptr()), 1, rep, flags))
torch.cuda.synchronize()
st = np.fromfile(path, np.uint64).reshape(-1, 8).astype(np.int64)
os.remove(path)
ok = st[:, 0] > 0
st = st[ok]
t0 = st[:, 0].min()
span = (st[:, 1].max() - t0) * 1e-3
dur = (st[:, 1] - st[:, 0]) * 1e-3
lines = info["lines"]
print(f"{cfgname}: {len(st)} tasks, {sweeps} sweeps, span {span:.1f} us ({span / sweeps / 1e3:.3f} ms/sweep), "
      f"executor {tracer.info()['executor']}, requirements {info['wave_requirements']}")
print(f"task duration mean {dur.mean():.1f} us (min {dur.min():.1f}, max {dur.max():.1f}); "
      f"tasks in flight (mean) {dur.sum() / span:.1f}; CTAs {len(np.unique(st[:, 6]))}")
for k, name in ((2, "ready-wait"), (3, "gather"), (4, "reduce"), (5, "store")):
    per_line = st[:, k] / lines * 1e-3
    print(f"  {name:10s} per line: mean {per_line.mean():.3f} us  p10 {np.percentile(per_line, 10):.3f}  "
          f"p90 {np.percentile(per_line, 90):.3f}")
# in-flight profile over time (10 bins)
edges = np.linspace(0, span, 11)
s0 = (st[:, 0] - t0) * 1e-3
s1 = (st[:, 1] - t0) * 1e-3
inflight = [((s0 < b) & (s1 > a)).sum() for a, b in zip(edges[:-1], edges[1:])]
print("  tasks overlapping each tenth of the span:", inflight)
# per (sweep, chunk): start-time lag between consecutive views, in lines
nch = Sp // min(32, Sp)
allst = np.fromfile(path, np.uint64) if os.path.exists(path) else None
per_sweep = info["views"] * nch
tick = np.nonzero(ok)[0]
start = dict(zip(tick.tolist(), st[:, 0].tolist()))
end = dict(zip(tick.tolist(), st[:, 1].tolist()))
lags = []
for tk in tick:
    v = (tk % per_sweep) // nch
    if v + 1 < info["views"] and tk + nch in start:
        lags.append((start[tk + nch] - start[tk]) * 1e-3)
lags = np.array(lags)
line_us = dur.mean() / lines
print(f"  view-to-view start lag: mean {lags.mean():.2f} us = {lags.mean() / line_us:.1f} lines of {line_us:.3f} us; "
      f"sweep = {info['views']} lags + one task = {(info['views'] * lags.mean() + dur.mean()) / 1e3:.3f} ms")
