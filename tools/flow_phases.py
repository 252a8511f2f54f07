"""Per-task phase times of the dataflow MART executor (diagnostics):
python tools/flow_phases.py c4  -> one sweep with USCG_SWEEP_PROFILE stamps,
then the mean time per phase (grab -> traced -> ready -> factor -> scattered
-> published) for single-warp updaters (P = 1), in microseconds."""
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
path = os.path.join(tempfile.mkdtemp(), "prof.bin")
os.environ["USCG_SWEEP_PROFILE"] = path
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2208_12964_b200 as ub  # noqa: E402
from paper_2208_12964_b200 import uscg, workloads  # noqa: E402

wl = workloads.make(sys.argv[1] if len(sys.argv) > 1 else "c4")
S = wl.problems
tracer = ub.Tracer(wl.geom, wl.spec, False)
truth = workloads.phantom_fields(wl, S).astype(np.float32)
proj = ub.project_stack(tracer, truth)
tracer.build_schedule()
info = tracer.info()
units = info["views"] * info["lines"]
Sp = ub.problem_stride(S)
pin = np.zeros((units, Sp), np.float32)
pin[:, :S] = proj.reshape(S, units).T
proj_d = torch.from_numpy(pin).cuda()
field_d = torch.ones((info["cell_count"], Sp), dtype=torch.float32, device="cuda")
L = ub.load()
flags = uscg.DEVICE_POINTERS | uscg.LAYOUT_INTERLEAVED
cfg = uscg._Cfg(wl.beta, 0.0, 1, 1.0, 0.0)
rep = (uscg._Report * S)()
uscg._check(L.uscg_reconstruct(tracer.h, uscg.C.c_void_p(proj_d.data_ptr()), S, uscg.C.byref(cfg),
                               uscg.C.c_void_p(field_d.data_ptr()), 1, rep, flags))
torch.cuda.synchronize()
st_all = np.fromfile(path, np.uint64).reshape(-1, 16).astype(np.int64)
os.remove(path)
ok = (st_all[:, 0] > 0) & (st_all[:, 6] > 0)
st = st_all[ok]
t0 = st[:, 0].min()
span = (st[:, 6].max() - t0) / 1e3
ph = {"metadata": (0, 9), "trace": (9, 8), "wait": (8, 1), "gather+sum": (2, 3), "factor": (3, 4), "scatter": (4, 5),
      "publish": (5, 6)}
print(f"{wl.name}: {len(st)} tasks, sweep {span:.0f} us, reconstruct {rep[0].seconds * 1e3:.1f} ms (profiled)")
for k, (a, b) in ph.items():
    d = (st[:, b] - st[:, a]) / 1e3
    print(f"  {k:11s} mean {d.mean():8.2f} us  p50 {np.median(d):8.2f}  p90 {np.percentile(d, 90):8.2f}")
cells = tracer.trace_counts().reshape(-1)
print(f"  cells/line mean {cells.mean():.0f} max {cells.max()}")

# ---- hand-offs: for each task that waited, the time from its binding
# predecessor's publish (stamp 6) to the end of its own spin (stamp 1) ----
sch = tracer.schedule()
order, pred_off, preds = sch["order"], sch["pred_off"].astype(np.int64), sch["preds"]
pos_of = np.empty(len(order), np.int64)
pos_of[order] = np.arange(len(order))
hops, waited = [], 0
n_tasks = len(order)
for pos in range(n_tasks):
    r = int(order[pos])
    a, b = pred_off[r], pred_off[r + 1]
    if a == b or st_all[pos, 1] == 0:
        continue
    pp = pos_of[preds[a:b]]
    pub = st_all[pp, 6]
    if (pub == 0).any():
        continue
    bind = pub.max()
    if st_all[pos, 1] - st_all[pos, 8] > 300:  # spun > 0.3 us: it waited on its predecessors
        waited += 1
        hops.append(st_all[pos, 1] - bind)
hops = np.array(hops) / 1e3
print(f"  tasks that waited: {waited} of {n_tasks}; hand-off (binding publish -> spin end) mean {hops.mean():.2f} us, "
      f"p50 {np.median(hops):.2f}, p90 {np.percentile(hops, 90):.2f}")
print(f"  levels per sweep {sch['levels']}: sweep / levels = {span / sch['levels']:.2f} us per level")
