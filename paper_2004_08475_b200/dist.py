"""Multi-GPU range partition: one process per GPU,
``torch.distributed`` over NCCL for the plumbing.

    idx = replicate_index(cells, scalars)          # rank 0 sorts, NCCL broadcast
    res = extract_isosurface_partitioned(idx, IsoParams(iso=0.0))
    res.fat           # this rank's slice of the global soup
    res.offset        # where it starts in the global (single-GPU) order
    res.total         # global triangle count

Why this is exact: the reference's output order is candidate order, owner
cell major (pipeline.cpp:40-57), and a CellId is a sorted position, so rank r
extracting cells [n*r/N, n*(r+1)/N) produces exactly the r-th contiguous
slice of the single-GPU output; an exclusive scan of the all-gathered
per-rank counts gives every slice its global offset.  The per-rank search
reads the whole replicated index (neighbours cross the range boundary),
which is why the index is replicated rather than partitioned.

The collective and extraction steps are plain functions of
(counts, ranges), so tests run the same logic over gloo on CPU with the
oracle standing in for the GPU extractor (tests/test_dist.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np


def cell_range(n: int, rank: int, world: int):
    """contiguous slice of the sorted cells owned by `rank`"""
    return n * rank // world, n * (rank + 1) // world


def exclusive_offsets(counts):
    """global start of each rank's slice (exclusive scan of the counts)"""
    off = np.zeros(len(counts) + 1, np.int64)
    np.cumsum(np.asarray(counts, np.int64), out=off[1:])
    return off


def allgather_counts(local: int, group=None, device=None):
    """all ranks' counts, in rank order"""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.tensor([int(local)], dtype=torch.int64, device=device)
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [int(x.item()) for x in out]


@dataclass
class PartitionedResult:
    fat: object          # this rank's triangles (or duals), candidate order
    offset: int          # global position of fat[0]
    total: int           # global count
    counts: list         # per-rank counts
    cell_range: tuple
    stats: object        # this rank's ExtractionStats
    counters: tuple      # global (accepted, missing, finer, lower_key)


def allreduce_counters(stats, group=None, device=None):
    import torch
    import torch.distributed as dist
    t = torch.tensor([stats.duals_accepted, stats.duals_missing_corner,
                      stats.duals_finer_corner, stats.duals_lower_key_corner],
                     dtype=torch.int64, device=device)
    dist.all_reduce(t, group=group)
    return tuple(int(x) for x in t.tolist())


def partitioned(n, extract_range, group=None, device=None):
    """Run extract_range(lo, hi) -> (items, stats) on this rank's slice and
    compute its global offset.  Pure plumbing: the GPU path passes the
    library's extraction, the CPU tests the oracle's."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = cell_range(n, rank, world)
    items, stats = extract_range(lo, hi)
    counts = allgather_counts(len(items), group, device)
    off = exclusive_offsets(counts)
    counters = allreduce_counters(stats, group, device)
    return PartitionedResult(items, int(off[rank]), int(off[-1]), counts, (lo, hi), stats,
                             counters)


def _cudart():
    for name in ("libcudart.so.12", "libcudart.so"):
        try:
            lib = C.CDLL(name)
            lib.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
            lib.cudaMemcpy.restype = C.c_int
            return lib
        except OSError:
            continue
    raise OSError("libcudart not found")


def replicate_index(cells=None, scalars=None, device=None, group=None, src=0, stream=None):
    """Rank `src` builds the index (pack + radix sort); its sorted keys and
    scalars (16 B/cell) are broadcast over NCCL; the other ranks adopt them
    (directory + level map only, no sort).  Returns this rank's CellIndex."""
    import torch
    import torch.distributed as dist
    from . import amrx as P
    rank = dist.get_rank(group)
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    idx = None
    meta = torch.zeros(17, dtype=torch.int64, device=dev)
    if rank == src:
        idx = P.build_index(cells, scalars, device=dev.index, stream=stream)
        meta[0] = len(idx)
        meta[1:] = torch.from_numpy(idx.geometry()).to(dev)
    dist.broadcast(meta, src, group=group)
    n = int(meta[0].item())
    geometry = meta[1:].cpu().numpy()
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    scal = torch.empty(n, dtype=torch.float64, device=dev)
    if rank == src:
        kp, sp = idx.device_arrays()
        rt = _cudart()
        torch.cuda.synchronize(dev)
        if rt.cudaMemcpy(keys.data_ptr(), kp, n * 8, 3) or \
                rt.cudaMemcpy(scal.data_ptr(), sp, n * 8, 3):
            raise RuntimeError("device copy failed")
    dist.broadcast(keys, src, group=group)
    dist.broadcast(scal, src, group=group)
    torch.cuda.synchronize(dev)
    if rank != src:
        idx = P.adopt_index(keys.data_ptr(), scal.data_ptr(), n, geometry, device=dev.index,
                            stream=stream)
    return idx


def extract_isosurface_partitioned(index, params, group=None, out=None, device=None):
    """this rank's slice of extract_isosurface + its global offset"""
    from . import amrx as P

    def run(lo, hi):
        r = P.extract_isosurface(index, params, cell_range=(lo, hi), out=out)
        return r.fat, r.stats

    return partitioned(len(index), run, group, device)


def extract_dual_mesh_partitioned(index, group=None, device=None):
    """this rank's slice of extract_dual_mesh + its global offset"""
    from . import amrx as P

    def run(lo, hi):
        d = P.extract_dual_mesh(index, cell_range=(lo, hi))
        return d, d.stats

    return partitioned(len(index), run, group, device)
