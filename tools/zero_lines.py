"""C2 diagnostics: how much of the wave executor's row traffic belongs to
lines whose measurements are zero for every problem of a 32-problem chunk
(lines the reference skips, solver.cpp:37-38)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2208_12964_b200 as ub
from paper_2208_12964_b200 import workloads

wl = workloads.make("c2")
S = wl.problems
tr = ub.Tracer(wl.geom, wl.spec, False)
truth = workloads.phantom_fields(wl, S)
proj = workloads.add_noise(wl, ub.project_stack(tr, truth.astype(np.float32))).astype(np.float32)
counts = tr.trace_counts().reshape(-1).astype(np.int64)
units = counts.size
nz = proj.reshape(S, units) != 0
L = wl.geom.det_u if hasattr(wl.geom, "det_u") else units // 90
print("units", units, "cells/line mean", counts.mean(), "nonempty lines", (counts > 0).sum())
for P in (32, 16, 8):
    ch = nz.reshape(S // P, P, units).any(axis=1)  # [chunks, units] line updates someone
    zero_cells = ((~ch) * counts[None, :]).sum()
    tot = counts.sum() * (S // P)
    print(f"P={P}: all-zero (chunk, line) pairs {(~ch & (counts > 0)[None, :]).sum()} of {(counts > 0).sum() * (S // P)}; "
          f"their cell visits {zero_cells / tot:.3f} of all")
per_line = (~nz.reshape(4, 32, units).any(axis=1)).reshape(4, 90, -1)
print("zero lines per view (chunk 0, first views):", per_line[0, :4].sum(axis=1))
v0 = per_line[0, 0]
print("zero pattern view 0 chunk 0 (first/last 80):", ''.join('0' if z else '1' for z in v0[:80]), ''.join('0' if z else '1' for z in v0[-80:]))
