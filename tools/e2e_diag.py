"""Where the batched end-to-end step spends its time (diagnostics): per-stack
solve time (reports) inside uscg_reconstruct_batch versus the whole call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2208_12964_b200 as ub  # noqa: E402
from paper_2208_12964_b200 import uscg, workloads  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 5
wl = workloads.make("c2")
S = wl.problems
ctx = ub.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
tr = ub.Tracer(wl.geom, wl.spec, False, ctx=ctx)
truth = workloads.phantom_fields(wl, S).astype(np.float32)
proj = ub.project_stack(tr, truth).reshape(S, -1)
tr.build_schedule()
cells = tr.info()["cell_count"]
stacks = [torch.from_numpy(proj.copy()).pin_memory() for _ in range(K)]
fields = [torch.empty((S, cells), dtype=torch.float32).pin_memory() for _ in range(K)]
L = ub.load()
cfg = uscg._Cfg(wl.beta, 0.0, 1, 1.0, 0.0)
reps = (uscg._Report * (K * S))()


def run(n, with_reps=True):
    pp = (uscg.C.c_void_p * n)(*[uscg.C.c_void_p(x.data_ptr()) for x in stacks[:n]])
    ff = (uscg.C.c_void_p * n)(*[uscg.C.c_void_p(x.data_ptr()) for x in fields[:n]])
    uscg._check(L.uscg_reconstruct_batch(tr.h, n, pp, S, uscg.C.byref(cfg), ff, 0, reps if with_reps else None, 0))


run(2)
torch.cuda.synchronize()
for with_reps in (False, True):
    t0 = time.perf_counter()
    run(K, with_reps)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    sol = [reps[b * S].seconds * 1e3 for b in range(K)] if with_reps else []
    print(f"K={K} reports={with_reps}: wall {wall:.2f} ms = {wall / K:.2f} ms/stack; solves (ms) "
          + " ".join(f"{x:.2f}" for x in sol))
# sequential one-call-per-stack through the device-pointer path for comparison
pd = torch.from_numpy(np.ascontiguousarray(proj.T)).cuda() if S > 1 else None
t0 = time.perf_counter()
for b in range(K):
    f = fields[b].numpy()
    uscg._check(L.uscg_reconstruct(tr.h, uscg.C.c_void_p(stacks[b].data_ptr()), S, uscg.C.byref(cfg),
                                   uscg.C.c_void_p(fields[b].data_ptr()), 0, reps, 0))
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
print(f"sequential host calls: {wall / K:.2f} ms/stack (solve {reps[0].seconds * 1e3:.2f} ms)")
