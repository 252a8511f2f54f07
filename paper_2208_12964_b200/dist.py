"""Multi-GPU plumbing (one process per GPU).

SURVEY.md §8(e): the 2D-stack configuration shards by slice with no
communication during iterations; the projector shards by view (every
(view, line) is independent and the field read-only,
proj/src/phantom.cpp:182-211); resampling shards by slice
(proj/src/phantom.cpp:149-163); the generator shards by detector row with one
exchange; cone-beam MART (C3/C4) does not shard (the reference's update
within a view is sequential), so it runs replicas only.
torch.distributed is used for rendezvous, the barrier around the timed region,
the max-over-ranks timing reduction and the optional end gather of fields —
never inside a sweep.
"""
from __future__ import annotations

import os
from typing import Tuple

import numpy as np


def env_rank() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block [lo, hi) of n items for `rank` (strong scaling of a
    fixed stack: slices [lo, hi) on this GPU)."""
    lo = n * rank // world
    hi = n * (rank + 1) // world
    return lo, hi


def rank_seed(base: int, rank: int) -> int:
    """Seed of rank `rank`'s own stack under weak scaling (distinct phantoms)."""
    return base + 1000 * rank


def max_over_ranks(values, device=None):
    """Element-wise max over ranks of a list of floats (the timing rule:
    a multi-GPU number is the slowest rank's device time)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def sum_over_ranks(values, device=None):
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(x) for x in t.cpu()]


def gather_stack(local: np.ndarray, n_total: int, rank: int, world: int, device=None):
    """End-of-run gather of slice-sharded fields to rank 0: local holds this
    rank's shard(n_total) rows; returns the (n_total, ...) stack on rank 0 and
    None elsewhere. One collective after the iterations, none during."""
    import torch
    import torch.distributed as dist
    lo, hi = shard(n_total, rank, world)
    assert local.shape[0] == hi - lo
    row = int(np.prod(local.shape[1:]))
    cap = (n_total + world - 1) // world
    buf = torch.zeros((cap, row), dtype=torch.float32, device=device)
    buf[: hi - lo] = torch.from_numpy(np.ascontiguousarray(local, dtype=np.float32).reshape(hi - lo, row)).to(buf)
    if world == 1:
        return buf[:n_total].cpu().numpy().reshape((n_total,) + local.shape[1:])
    parts = [torch.zeros_like(buf) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, parts, dst=0)
    if rank != 0:
        return None
    rows = [parts[r][: shard(n_total, r, world)[1] - shard(n_total, r, world)[0]] for r in range(world)]
    return torch.cat(rows).cpu().numpy().reshape((n_total,) + local.shape[1:])


# ---------------------------------------------------------------------------
# row-sharded first-view generator (generator row)
# ---------------------------------------------------------------------------


def concat_caches(parts):
    """Concatenate record stores of consecutive line blocks, in block order:
    parts = [(offsets, phi_a, phi_b, keys), ...] (torch tensors; offsets local,
    starting at 0, as int32 bit patterns of u32). Returns the full store."""
    import torch
    dev = parts[0][0].device
    base = 0
    offs, pas, pbs, keys = [], [], [], []
    for off, pa, pb, key in parts:
        L = off.numel() - 1
        offs.append(off[:L].to(torch.int64) + base)
        pas.append(pa)
        pbs.append(pb)
        keys.append(key)
        base += pa.numel()
    offs.append(torch.tensor([base], dtype=torch.int64, device=dev))
    if base >= 1 << 32:
        raise ValueError("record count must fit in 32 bits")
    full_off = torch.cat(offs)
    full_off = torch.where(full_off >= 1 << 31, full_off - (1 << 32), full_off).to(torch.int32)  # u32 bits
    return full_off, torch.cat(pas), torch.cat(pbs), torch.cat(keys)


def assemble_cache(off, pa, pb, key):
    """The generator's one exchange: every rank holds the records of a
    contiguous block of lines; all ranks receive the full store. All-gather of
    the per-rank (lines, records) counts, then one all-gather per array of the
    segments padded to the largest (NCCL on the GPU, gloo on the CPU), and the
    record bases from an exclusive scan of the counts (concat_caches)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return off, pa, pb, key
    world = dist.get_world_size()
    dev = off.device
    counts = torch.tensor([off.numel() - 1, pa.numel()], dtype=torch.int64, device=dev)
    allc = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(allc, counts)
    Ls = [int(c[0]) for c in allc]
    Rs = [int(c[1]) for c in allc]

    def gather(t, n, m):
        pad = torch.zeros(max(m, 1), dtype=t.dtype, device=dev)
        pad[:n] = t[:n]
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad)
        return parts

    offp = gather(off, Ls[dist.get_rank()] + 1, max(Ls) + 1)
    pap = gather(pa, pa.numel(), max(Rs))
    pbp = gather(pb, pb.numel(), max(Rs))
    kp = gather(key, key.numel(), max(Rs))
    return concat_caches([(offp[r][: Ls[r] + 1], pap[r][: Rs[r]], pbp[r][: Rs[r]], kp[r][: Rs[r]])
                          for r in range(world)])


def generate_sharded(spec, geom, rank: int, world: int, ctx=None):
    """Rank `rank` generates the first-view records of detector rows
    shard(det_v) and every rank assembles the full tracer (assemble_cache)."""
    from .uscg import Tracer
    src, det = geom.first_view_rays()
    r0, r1 = shard(geom.det_v, rank, world)
    l0, l1 = r0 * geom.det_u, r1 * geom.det_u
    local = Tracer.from_rays(spec, src[l0:l1], det[l0:l1], 1, ctx=ctx)
    part = local.copy_cache(device=True)
    local.close()
    full = assemble_cache(*part)
    return Tracer.from_key_cache(spec, *full, geom.views, geom.view_angles, geom=geom, ctx=ctx)


# ---------------------------------------------------------------------------
# view-sharded projector (projector row)
# ---------------------------------------------------------------------------


def view_subset_tracer(tracer, v0: int, v1: int):
    """A tracer over views [v0, v1) of `tracer`, sharing its record store (the
    symmetry-compressed store is view-independent: a copy of the one-view
    records on the same device, no regeneration)."""
    import dataclasses

    from .uscg import Tracer
    th = np.asarray(tracer.geom.thetas(), dtype=np.float64)[v0:v1]
    off, pa, pb, key = tracer.copy_cache(device=True)
    geom = dataclasses.replace(tracer.geom, views=v1 - v0, view_angles=th)
    return Tracer.from_key_cache(tracer.spec, off, pa, pb, key, v1 - v0, th, geom=geom, ctx=tracer.ctx)


def project_views_local(tracer, fields: np.ndarray, rank: int, world: int) -> np.ndarray:
    """This rank's share of generate_projections: the binary projections of
    every field over views shard(views, rank, world): (S, v1 - v0, lines)."""
    from .uscg import project_stack
    v0, v1 = shard(tracer.info()["views"], rank, world)
    if v1 == v0:
        return np.zeros((fields.shape[0], 0, tracer.info()["lines"]), np.float32)
    sub = view_subset_tracer(tracer, v0, v1)
    try:
        return project_stack(sub, fields)
    finally:
        sub.close()


def concat_views(parts) -> np.ndarray:
    """The rank-ordered view blocks (each (S, views_r, lines)) as one stack."""
    return np.concatenate(list(parts), axis=1)


def all_gather_views(local: np.ndarray, n_views: int, rank: int, world: int, device=None) -> np.ndarray:
    """Every rank receives the full (S, n_views, lines) projections: one
    all-gather of the view blocks padded to the largest shard."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    S, _, lines = local.shape
    cap = (n_views + world - 1) // world
    buf = torch.zeros((S, cap, lines), dtype=torch.float32, device=device)
    lo, hi = shard(n_views, rank, world)
    buf[:, : hi - lo] = torch.from_numpy(np.ascontiguousarray(local, dtype=np.float32)).to(buf)
    parts = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    return concat_views([parts[r][:, : shard(n_views, r, world)[1] - shard(n_views, r, world)[0]].cpu().numpy()
                         for r in range(world)])


def project_view_sharded(tracer, fields: np.ndarray, rank: int, world: int, device=None) -> np.ndarray:
    """generate_projections on N GPUs: each rank projects its view block, one
    all-gather assembles the full set on every rank."""
    local = project_views_local(tracer, fields, rank, world)
    return all_gather_views(local, tracer.info()["views"], rank, world, device)


# ---------------------------------------------------------------------------
# slice-sharded resampling (resample row)
# ---------------------------------------------------------------------------


def slice_subgrid(spec, s0: int, s1: int):
    """The grid of slices [s0, s1) of a volume grid (same rings, sector law,
    slice height)."""
    from .uscg import GridSpec
    return GridSpec(spec.n, spec.ring_spacing, spec.slice_height, spec.mode, ring_counts=spec.ring_counts,
                    n_slices=s1 - s0)


def resample_local(spec, field: np.ndarray, npix: int, rank: int, world: int, ctx=None) -> np.ndarray:
    """field_to_cartesian of this rank's slices shard(slices, rank, world) of
    one volume field (reference flat order): (s1 - s0, npix, npix)."""
    from .uscg import resample_stack
    s0, s1 = shard(spec.slices(), rank, world)
    cps = spec.cells_per_slice()
    if s1 == s0:
        return np.zeros((0, npix, npix), np.float32)
    sub = slice_subgrid(spec, s0, s1)
    return resample_stack(sub, np.asarray(field).reshape(-1)[s0 * cps: s1 * cps][None], npix, ctx)[0]
