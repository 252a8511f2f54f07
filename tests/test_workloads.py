"""Synthetic BASELINE workloads and the bench harness on the CPU."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_workload_shapes_match_baseline_configs():
    from paper_2208_12964_b200 import workloads
    c1 = workloads.make("c1")
    assert c1.spec.cell_count() == 12868 and c1.geom.det_u == 128 and c1.geom.views == 36
    assert c1.geom.thetas()[-1] == 175.0  # 36 views over 180 degrees
    c2 = workloads.make("c2")
    assert c2.spec.cells_per_slice() == 205888 and c2.problems == 128 and c2.geom.views == 90
    c3 = workloads.make("c3")
    assert c3.spec.cell_count() == 6588416 and c3.geom.lines() == 65536
    c4 = workloads.make("c4")
    assert c4.spec.cell_count() == 52707328
    c5 = workloads.make("c5")
    assert c5.spec.cells_per_slice() == 823550 and c5.geom.lines() == 1024 * 1024


def test_phantoms_are_seeded_and_in_range():
    from paper_2208_12964_b200 import workloads
    wl = workloads.make("c1")
    a = workloads.phantom_fields(wl, 2)
    b = workloads.phantom_fields(wl, 2)
    assert np.array_equal(a, b)
    assert not np.array_equal(a[0], a[1])
    assert a.min() >= 0 and a.max() > 0.1
    lump = workloads.make("c4")
    x, y, z = workloads.cell_centroids(workloads.make("c1").spec)
    v = workloads.lump_value(np.random.default_rng(0), x, y, 0.0)
    assert set(np.unique(v)) <= {0.0, 0.2, 8.0}
    assert lump.noise == "poisson"


def test_noise_is_multiplicative_and_clipped():
    from paper_2208_12964_b200 import workloads
    wl = workloads.make("c2")
    p = np.ones((4, 100), np.float32)
    p[0] = 0
    q = workloads.add_noise(wl, p)
    assert np.all(q[0] == 0) and np.all(q >= 0)
    assert 0.005 < np.std(q[1:]) < 0.02


@pytest.mark.timeout(600)
def test_bench_reference_arm_prints_one_json_line():
    """bench.py --impl reference: the CPU arm (oracle port on the verbatim
    config) keeps the JSON contract, sized to finish in seconds here."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--config", "c1"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0
