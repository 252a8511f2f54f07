"""bench.py's multi-rank C2 logic on one GPU: every rank's share is run by the
same bench_mart call a rank makes (no process group: the collectives reduce
over one process), so the sharded and weak-scaling paths the driver's
N-GPU run takes are exercised here; the JSON contract of the line holds."""
import argparse
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _args(**kw):
    a = dict(gpus=1, steps=2, warmup=1, config="c2", problems=8, impl="ours", no_cpu=True, no_e2e=False,
             no_uscg=True, no_store_fed=True, no_weak=False)
    a.update(kw)
    return argparse.Namespace(**a)


def test_bench_mart_rank_shares_and_weak_path(ub):
    sys.path.insert(0, ROOT)
    import bench
    gpu = bench.Gpu(0)
    args = _args()
    # rank 1 of 2 reconstructs its shard and returns nothing
    assert bench.bench_mart(gpu, "c2", args, 1, 2, cpu=False, iso=False) is None
    # rank 0 of 2: its shard; the line carries the contract's keys
    line = bench.bench_mart(gpu, "c2", args, 0, 2, cpu=False, iso=False)
    assert line["per_gpu_slices"] == 4 and line["n_gpus"] == 2 and line["scaling"] == "strong"
    for k in ("metric", "value", "unit", "ms_per_step", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in line
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["gpu_launches"] > 0
    # the weak-scaling extra: a whole stack on this rank
    weak = bench.bench_mart(gpu, "c2", args, 0, 2, cpu=False, e2e=False, iso=False, weak=True)
    assert weak["per_gpu_slices"] == 8 and weak["value"] > 0
