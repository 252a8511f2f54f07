"""Multi-rank host logic of the slice-stack path, world_size 2 over gloo on
the CPU (the GPU pool runs one GPU per call).

Each rank reconstructs its own shard of a slice stack with the CPU oracle
(the per-rank work of the sharded device path), the fields are gathered to
rank 0 once at the end, and the result must equal the single-process run;
the timing reduction is the max over ranks.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stack_inputs(S):
    import oracle
    orc = oracle.Orc()
    grid = oracle.OrcGrid(16, 1 / 16, 1, 1 / 16, False, orc.ring_counts_m1(16))
    s, d = orc.rays_arc((-3, 0, 0), (1.5, 0, 0), 48, 38.94 / 48)
    oc = orc.cache(grid, s, d)
    th = np.array([12.0 * i for i in range(30)])
    truth = np.random.default_rng(5).uniform(0.2, 2.0, (S, grid.cell_count()))
    proj = np.stack([oc.project(th, truth[p]) for p in range(S)])
    return oc, th, proj


def _worker(rank, world, port, S, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    from paper_2208_12964_b200 import dist as udist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    oc, th, proj = _stack_inputs(S)
    lo, hi = udist.shard(S, rank, world)
    local = np.stack([oc.reconstruct(th, proj[p], beta=0.5, tolerance=0, max_sweeps=3)[0] for p in range(lo, hi)])
    stack = udist.gather_stack(local, S, rank, world)
    t = udist.max_over_ranks([1.0 + rank, 5.0 - rank])
    tot = udist.sum_over_ranks([hi - lo])
    dist.barrier()
    if rank == 0:
        np.save(os.path.join(out_dir, "stack.npy"), stack)
        np.save(os.path.join(out_dir, "red.npy"), np.array(t + tot))
    dist.destroy_process_group()


def test_shard_covers_stack_exactly_once():
    from paper_2208_12964_b200.dist import shard
    for S in (1, 7, 128):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                lo, hi = shard(S, r, world)
                seen += list(range(lo, hi))
            assert seen == list(range(S))


def test_rank_seeds_distinct():
    from paper_2208_12964_b200.dist import rank_seed
    assert len({rank_seed(12345, r) for r in range(8)}) == 8


@pytest.mark.timeout(300)
def test_two_rank_slice_sharding_matches_single_process(tmp_path):
    S = 5
    port = _free_port()
    mp.spawn(_worker, args=(2, port, S, str(tmp_path)), nprocs=2, join=True)
    stack = np.load(tmp_path / "stack.npy")
    red = np.load(tmp_path / "red.npy")
    oc, th, proj = _stack_inputs(S)
    want = np.stack([oc.reconstruct(th, proj[p], beta=0.5, tolerance=0, max_sweeps=3)[0] for p in range(S)])
    assert np.array_equal(stack, want.astype(np.float32))
    assert list(red[:2]) == [2.0, 5.0]     # max over ranks
    assert red[2] == S                      # every slice reconstructed once


# ---------------------------------------------------------------------------
# row-sharded generator: the exchange (generator row)
# ---------------------------------------------------------------------------


def _cone_rays():
    import oracle
    orc = oracle.Orc()
    grid = oracle.OrcGrid.reference(12, True)
    # 5 x 7 flat panel: the row blocks of two ranks are uneven
    s, d = orc.rays_flat((-3, 0, 0), (10, 0, 0), 5, 7, 1.0, 1.0)
    return orc, grid, s, d


def _key_layout(oc):
    """record store of an oracle cache in the device layout (keys without flags)"""
    import torch
    rec = oc.records
    keys = rec["ring"].astype(np.uint32) | (rec["slice"].astype(np.uint32) << 12)
    return (torch.from_numpy(oc.offsets.astype(np.uint32).view(np.int32).copy()),
            torch.from_numpy(rec["phi_a"].copy()), torch.from_numpy(rec["phi_b"].copy()),
            torch.from_numpy(keys.view(np.int32).copy()))


def _gen_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_2208_12964_b200 import dist as udist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc, grid, s, d = _cone_rays()
    r0, r1 = udist.shard(7, rank, world)
    part = _key_layout(orc.cache(grid, s[r0 * 5:r1 * 5], d[r0 * 5:r1 * 5]))
    full = udist.assemble_cache(*part)
    dist.barrier()
    if rank == 0:
        np.savez(os.path.join(out_dir, "full.npz"), *[t.numpy() for t in full])
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_generator_exchange_assembles_the_full_store(tmp_path):
    port = _free_port()
    mp.spawn(_gen_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    got = np.load(tmp_path / "full.npz")
    orc, grid, s, d = _cone_rays()
    want = [t.numpy() for t in _key_layout(orc.cache(grid, s, d))]
    for k, w in enumerate(want):
        assert np.array_equal(got[f"arr_{k}"], w), k


# ---------------------------------------------------------------------------
# the slice-sharded bench inputs, the view-sharded projector's exchange and the
# slice-sharded resample
# ---------------------------------------------------------------------------


def test_sharded_stack_inputs_are_rows_of_the_full_stack():
    """bench.py's C2 shards generate exactly their rows of the full stack's
    phantoms and noise (problem p seeded by p, whatever the shard)."""
    from paper_2208_12964_b200 import workloads
    from paper_2208_12964_b200.dist import shard
    wl = workloads.make("c2", problems=5)
    full = workloads.phantom_fields(wl, 5)
    proj = np.random.default_rng(1).uniform(0, 2, (5, 40)).astype(np.float32)
    noisy = workloads.add_noise(wl, proj)
    for world in (2, 3):
        for r in range(world):
            lo, hi = shard(5, r, world)
            assert np.array_equal(workloads.phantom_fields(wl, hi - lo, first=lo), full[lo:hi])
            assert np.array_equal(workloads.add_noise(wl, proj[lo:hi], first=lo), noisy[lo:hi])


def _view_case():
    import oracle
    orc = oracle.Orc()
    grid = oracle.OrcGrid(16, 1 / 16, 1, 1 / 16, False, orc.ring_counts_m1(16))
    s, d = orc.rays_arc((-3, 0, 0), (1.5, 0, 0), 48, 38.94 / 48)
    th = np.array([360.0 * i / 11 for i in range(11)])
    truth = np.random.default_rng(8).uniform(0.2, 2.0, (3, grid.cell_count()))
    return orc, grid, s, d, th, truth


def _view_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_2208_12964_b200 import dist as udist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc, grid, s, d, th, truth = _view_case()
    v0, v1 = udist.shard(th.size, rank, world)
    oc = orc.cache(grid, s, d)
    local = np.stack([oc.project(th[v0:v1], truth[p]) for p in range(truth.shape[0])]).astype(np.float32)
    full = udist.all_gather_views(local, th.size, rank, world)
    np.save(os.path.join(out_dir, f"views{rank}.npy"), full)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_view_sharded_projection_exchange(tmp_path):
    """Each rank projects its view block; one all-gather gives every rank the
    full projection set (the per-rank projections here are the oracle's, the
    stand-in for each GPU's project_views_local)."""
    port = _free_port()
    mp.spawn(_view_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    orc, grid, s, d, th, truth = _view_case()
    oc = orc.cache(grid, s, d)
    want = np.stack([oc.project(th, truth[p]) for p in range(truth.shape[0])]).astype(np.float32)
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"views{r}.npy"), want)


def _res_case():
    import oracle
    orc = oracle.Orc()
    grid = oracle.OrcGrid(12, 1 / 12, 10, 2 / 12, True, orc.ring_counts_m1(12))
    field = np.random.default_rng(4).uniform(0, 1, grid.cell_count())
    return orc, grid, field


def _res_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    import torch.distributed as dist
    from paper_2208_12964_b200 import dist as udist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc, grid, field = _res_case()
    s0, s1 = udist.shard(grid.n_slices, rank, world)
    cps = grid.cells_per_slice()
    sub = oracle.OrcGrid(grid.n_rings, grid.ring_spacing, s1 - s0, grid.slice_height, True, grid.counts)
    local = orc.field_to_cartesian(sub, field[s0 * cps:s1 * cps], 32).astype(np.float32)
    stack = udist.gather_stack(local, grid.n_slices, rank, world)
    if rank == 0:
        np.save(os.path.join(out_dir, "img.npy"), stack)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_slice_sharded_resample(tmp_path):
    """Each rank resamples its slices (the oracle's field_to_cartesian on the
    rank's sub-volume, the stand-in for dist.resample_local), rank 0 gathers
    the raster stack; it equals the single-process resample."""
    port = _free_port()
    mp.spawn(_res_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    orc, grid, field = _res_case()
    want = orc.field_to_cartesian(grid, field, 32).astype(np.float32)
    assert np.array_equal(np.load(tmp_path / "img.npy"), want)
