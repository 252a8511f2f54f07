"""Run levels of the dataflow schedule per run length: USCG_RUN=<n> python tools/levels_probe.py c3 [c4]"""
import os, sys
sys.path.insert(0, os.getcwd())
import paper_2208_12964_b200 as ub
from paper_2208_12964_b200 import workloads
for cfg in (sys.argv[1:] or ["c3"]):
    wl = workloads.make(cfg)
    tr = ub.Tracer(wl.geom, wl.spec, False)
    lv = tr.build_schedule()
    inf = tr.info()
    print(cfg, "run", os.environ.get("USCG_RUN"), "levels", lv, "max_cells", inf["max_line_cells"], "lines", inf["lines"], "views", inf["views"], flush=True)
