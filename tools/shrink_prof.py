"""Keep the per-task stamp columns the critical-chain analysis reads
(grab, start, end, publish, staged, deps-seen) of a USCG_SWEEP_PROFILE dump."""
import sys

import numpy as np

a = np.fromfile(sys.argv[1], np.uint64).reshape(-1, 16)
np.save(sys.argv[2], a[:, [0, 2, 5, 6, 7, 15]])
