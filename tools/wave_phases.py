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
problems = int(sys.argv[3]) if len(sys.argv) > 3 else None
wl = workloads.make(cfgname, problems=problems)
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
lines = info["lines"]
rec = 8 + 2 * lines
raw = np.fromfile(path, np.uint64).reshape(-1, rec).astype(np.int64)
os.remove(path)
st = raw[:, :8]
pub_all = raw[:, 8:8 + lines]
rdy_all = raw[:, 8 + lines:]
ok = st[:, 0] > 0
st = st[ok]
t0 = st[:, 0].min()
span = (st[:, 1].max() - t0) * 1e-3
dur = (st[:, 1] - st[:, 0]) * 1e-3
lines = info["lines"]
print(f"{cfgname} S={S}: {len(st)} tasks, {sweeps} sweeps, span {span:.1f} us ({span / sweeps / 1e3:.3f} ms/sweep), "
      f"executor {tracer.info()['executor']} ({tracer.info()['wave_ctas']} CTAs a task), "
      f"requirements {info['wave_requirements']}")
print(f"task duration mean {dur.mean():.1f} us (min {dur.min():.1f}, max {dur.max():.1f}); "
      f"tasks in flight (mean) {dur.sum() / span:.1f}; CTAs {len(np.unique(st[:, 6]))}")
for k, name in ((2, "ready-wait"), (3, "start->A"), (7, " copy-wait"), (4, "A->B"), (5, "B->C")):
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
P = int(os.environ.get("USCG_CHUNK_WIDTH", 32 if Sp > 64 else 16))
P = min(P, Sp)
nch = Sp // P
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

# ---- per-line chain analysis: what each line waited for ----
wa = tracer.wave_arrays()
dep_off = wa["dep_off"].astype(np.int64)
deps = wa["deps"].reshape(-1, 2).astype(np.int64)
V = info["views"]
hops, waits, periods, local = [], [], [], 0
ntk = raw.shape[0]
for tk in range(ntk):
    if st[tk, 0] == 0:
        continue
    sw, v, ch = tk // per_sweep, (tk % per_sweep) // nch, tk % nch
    pub, rdy = pub_all[tk], rdy_all[tk]
    periods.append(np.diff(pub[pub > 0]))
    for j in range(1, lines):
        u = v * lines + j
        best = 0
        for k in range(dep_off[u], dep_off[u + 1]):
            w, need = deps[k]
            xs, ov = w >> 31, w & 0x7FFFFFFF
            psw = sw - xs
            if psw < 0:
                continue
            ptk = psw * per_sweep + ov * nch + ch
            if ptk >= ntk or st[ptk, 0] == 0:
                continue
            best = max(best, pub_all[ptk, need - 1])
        if best and rdy[j] > 0:
            hops.append(rdy[j] - best)
            # line j became ready after line j-1 was published: it waited on another view
            waits.append(max(0, rdy[j] - pub[j - 1]))
hops = np.array(hops) * 1e-3
waits = np.array(waits) * 1e-3
per = np.concatenate(periods) * 1e-3
print(f"  line period (publish to publish) mean {per.mean():.3f} us, p50 {np.median(per):.3f}, p90 {np.percentile(per, 90):.3f}")
print(f"  consumer discovery (ready - binding publish): mean {hops.mean():.3f} us, p50 {np.median(hops):.3f}, "
      f"p90 {np.percentile(hops, 90):.3f} over {hops.size} lines with requirements")
print(f"  lines ready only after their predecessor's publish: {(waits > 0).mean():.3f}, mean excess {waits[waits > 0].mean():.3f} us")
