"""Schedule-build time per BASELINE configuration (diagnostics):
python tools/sched_time.py c2 c3 c4  (USCG_FLOW_VERBOSE=1 prints the phases)."""
import sys
import time

sys.path.insert(0, ".")
from paper_2208_12964_b200 import uscg as ub, workloads  # noqa: E402

for name in sys.argv[1:] or ["c2", "c3", "c4"]:
    wl = workloads.make(name)
    t0 = time.perf_counter()
    tr = ub.Tracer(wl.geom, wl.spec, False)
    t1 = time.perf_counter()
    levels = tr.build_schedule()
    t2 = time.perf_counter()
    print(f"{name}: tracer {t1 - t0:.2f} s, schedule {t2 - t1:.2f} s, levels {levels}", flush=True)
