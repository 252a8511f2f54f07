"""Profiling driver: C2 stack setup, one K2 projector call and one K3 MART
sweep on device-resident data (for ncu; never a bench number)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2208_12964_b200 as ub  # noqa: E402
from paper_2208_12964_b200 import uscg, workloads  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = workloads.make(cfgname, problems=int(sys.argv[2]) if len(sys.argv) > 2 else None)
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
out_d = torch.empty((units, Sp), dtype=torch.float32, device="cuda")
L = ub.load()
flags = uscg.DEVICE_POINTERS | uscg.LAYOUT_INTERLEAVED
uscg._check(L.uscg_project(tracer.h, uscg.C.c_void_p(field_d.data_ptr()), S, uscg.C.c_void_p(out_d.data_ptr()), flags))
cfg = uscg._Cfg(wl.beta, 0.0, 1, 1.0, 0.0)
rep = (uscg._Report * S)()
uscg._check(L.uscg_reconstruct(tracer.h, uscg.C.c_void_p(proj_d.data_ptr()), S, uscg.C.byref(cfg),
                               uscg.C.c_void_p(field_d.data_ptr()), 1, rep, flags))
torch.cuda.synchronize()
print("profile driver ok", info["levels"], rep[0].seconds)
