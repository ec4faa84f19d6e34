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
    out = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, t, group=group)
    return out.tolist()  # one host sync


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


# ---------------------------------------------------------------------------
# Distributed build (every rank holds a slice of the cell list).  The plan is
# pure integer arithmetic over packed keys, so tests run it over gloo on CPU.

def geometry_layout(geometry):
    """(major_shift, finest, coarsest, key_bits) from geometry word 15"""
    w = int(geometry[15])
    return w & 0xFF, (w >> 8) & 0xFF, (w >> 16) & 0xFF, (w >> 24) & 0xFF


def choose_splitters(samples, world):
    """world-1 strictly increasing key boundaries from the sorted union of
    every rank's evenly spaced samples; rank q owns keys [s_q, s_q+1) with
    s_0 = 0 and s_world = 2^63.  Negative samples (an empty slice's
    placeholders) are ignored, so empty slices do not pull splitters down."""
    import torch
    smp = torch.sort(samples.reshape(-1)).values.tolist()  # one host sync
    smp = [x for x in smp if x >= 0] or [0]
    cut = [smp[(len(smp) * q) // world] for q in range(1, world)]
    out = [0]
    for c in cut:
        out.append(max(int(c), out[-1] + 1))
    out.append(1 << 63)
    return out


def halo_ranges(bounds, geometry):
    """key range each rank must hold to extract its owned range exactly:
    its owned keys plus every key whose major coordinate (the most
    significant field of the key, i unless that axis is constant) lies
    within two coarsest cell widths -- a stencil point is within one owner
    width of its cell, and a cell containing it within one coarsest width
    of the point"""
    msh, finest, coarsest, bits = geometry_layout(geometry)
    hw = 2 << (coarsest - finest)  # two coarsest widths in packed units
    top = 1 << bits
    world = len(bounds) - 1
    lo, hi = [], []
    for q in range(world):
        a, b = bounds[q], min(bounds[q + 1], top)
        if b <= a:
            lo.append(a)
            hi.append(a)
            continue
        lo.append(max(0, (a >> msh) - hw) << msh)
        hi.append(min(top, ((b - 1) >> msh) + hw + 1 << msh))
    return lo, hi


def send_plan(sorted_keys, lo, hi):
    """(start, count) of the sorted local keys each rank needs"""
    import torch
    bl = torch.tensor(lo, dtype=sorted_keys.dtype, device=sorted_keys.device)
    bh = torch.tensor(hi, dtype=sorted_keys.dtype, device=sorted_keys.device)
    a = torch.searchsorted(sorted_keys, bl)
    b = torch.searchsorted(sorted_keys, bh)
    start, count = torch.stack([a, b - a]).tolist()  # one host sync
    return start, count


def global_geometry(bounds10, counts):
    """geometry words 0-10 from every rank's amrx_bounds output + count"""
    b = np.asarray(bounds10, np.int64).reshape(-1, 10)
    g = np.zeros(16, np.int64)
    g[0:3] = b[:, 0:3].min(0)
    g[3:9] = b[:, 3:9].max(0)
    m = 0
    for x in b[:, 9]:
        m |= int(x)
    g[9] = m
    g[10] = int(np.sum(np.asarray(counts, np.int64)))
    return g


def owned_split(rkeys, bounds, rank):
    """(keys below the owned range, keys in it) among a rank's received keys"""
    import torch
    s_r, s_r1 = bounds[rank], bounds[rank + 1]
    inside = rkeys >= s_r
    if s_r1 < (1 << 63):
        inside &= rkeys < s_r1
    below, own = torch.stack([(rkeys < s_r).sum(), inside.sum()]).tolist()  # one host sync
    return below, own


def exchange_runs(keys, scal, lo, hi, group=None, device=None):
    """send every rank the slice of my sorted (keys, scalars) inside its
    [lo, hi) (halos overlap, so some keys go to two ranks); returns what I
    received: `world` sorted runs, concatenated in rank order"""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    start, count = send_plan(keys, lo, hi)
    send = torch.cat([torch.stack([keys[a:a + c], scal[a:a + c].view(torch.int64)], 1)
                      for a, c in zip(start, count)])
    rc = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_to_all_single(rc, torch.tensor(count, dtype=torch.int64, device=device),
                           group=group)
    rcount = rc.tolist()
    recv = torch.empty((sum(rcount), 2), dtype=torch.int64, device=device)
    dist.all_to_all_single(recv, send, output_split_sizes=rcount, input_split_sizes=count,
                           group=group)
    return recv[:, 0].contiguous(), recv[:, 1].contiguous().view(torch.float64)


@dataclass
class DistributedIndex:
    index: object        # this rank's partition (CellIndex), global ids
    owned: tuple         # local position range of the cells this rank owns
    id_base: int         # global CellId of local position 0
    total: int           # global cell count
    seconds: dict        # host wall time per phase


class _DeviceArray:
    """a zero-copy view of library-owned device memory for torch
    (__cuda_array_interface__); `owner` keeps the memory alive"""

    def __init__(self, ptr, n, typestr, owner):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}
        self.owner = owner


def sorted_arrays(index, device):
    """torch views (no copy) of an index's sorted packed keys (int64) and
    scalars; valid only while `index` stays open (close it after the last
    use of the views)"""
    import torch
    n = len(index)
    kp, sp = index.device_arrays()
    keys = torch.as_tensor(_DeviceArray(kp, n, "<i8", index), device=device)
    scal = torch.as_tensor(_DeviceArray(sp, n, "<f8", index), device=device)
    return keys, scal


def build_distributed(cells, scalars, group=None, device=None, stream=None, samples=4096):
    """Distributed build_index: rank r holds a slice (cells, scalars) of the
    global cell list.  (1) bounds all-reduced into the global key geometry;
    (2) each rank radix-sorts its slice (amrx_index_sort_part); (3) sampled
    splitters give every rank a contiguous owned key range, widened by a
    halo of two coarsest cell widths; (4) one all-to-all moves each sorted
    run to the ranks whose ranges cover it; (5) each rank sorts what it
    received and indexes it (amrx_index_from_keys) with the global id of its
    first key.  Extracting the owned range then reproduces exactly the
    single-GPU slice of the output (candidate order is owner-cell major)."""
    import time
    import torch
    import torch.distributed as dist
    from . import amrx as P
    t0 = time.perf_counter()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    sh = stream.cuda_stream if stream is not None and hasattr(stream, "cuda_stream") else stream
    n_loc = cells.shape[0]
    b = torch.tensor(np.append(P.cell_bounds(cells, device=dev.index, stream=sh), n_loc),
                     dtype=torch.int64, device=dev)
    allb = torch.empty((world, 11), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allb, b, group=group)
    allb = allb.cpu().numpy()  # the geometry is host input to the sort
    g = global_geometry(allb[:, :10], allb[:, 10])
    n = int(g[10])
    t1 = time.perf_counter()
    part = P.sort_part(cells, scalars, g, device=dev.index, stream=sh)
    g = part.geometry()
    g[10] = n
    if geometry_layout(g)[3] > 63:
        raise P.UnsupportedError("distributed build needs keys of at most 63 bits")
    keys, scal = sorted_arrays(part, dev)  # views: `part` stays open until the exchange
    t2 = time.perf_counter()
    # splitters from evenly spaced samples of every rank's sorted slice
    pos = torch.linspace(0, max(n_loc - 1, 0), samples, device=dev).round().long()
    smp = keys[pos] if n_loc else torch.full((samples,), -1, dtype=torch.int64, device=dev)
    gathered = torch.empty(world * samples, dtype=smp.dtype, device=dev)
    dist.all_gather_into_tensor(gathered, smp.contiguous(), group=group)
    bounds = choose_splitters(gathered, world)
    lo, hi = halo_ranges(bounds, g)
    rkeys, rscal = exchange_runs(keys, scal, lo, hi, group, dev)
    del keys, scal
    part.close()
    t3 = time.perf_counter()
    below, own = owned_split(rkeys, bounds, rank)
    owns = allgather_counts(own, group, dev)
    id_base = int(sum(owns[:rank])) - below
    g[12], g[13], g[14] = id_base, lo[rank], hi[rank]
    index = None
    if len(rkeys) and own:
        index = P.index_from_keys(rkeys.data_ptr(), rscal.data_ptr(), len(rkeys), g,
                                  device=dev.index, stream=sh)
    t4 = time.perf_counter()
    return DistributedIndex(index, (below, below + own), id_base, n,
                            {"geometry": t1 - t0, "sort": t2 - t1, "exchange": t3 - t2,
                             "index": t4 - t3})


def extract_isosurface_distributed(dindex, params, group=None, out=None, device=None):
    """this rank's slice of extract_isosurface over a distributed index"""
    from . import amrx as P

    def run(lo, hi):
        if dindex.index is None or hi <= lo:
            return np.zeros((0, 9)), P.ExtractionStats()
        r = P.extract_isosurface(dindex.index, params, cell_range=(lo, hi), out=out)
        return r.fat, r.stats

    return partitioned_range(dindex.owned, run, group, device)


def extract_dual_mesh_distributed(dindex, group=None, device=None):
    """this rank's slice of extract_dual_mesh (global CellIds)"""
    from . import amrx as P

    def run(lo, hi):
        if dindex.index is None or hi <= lo:
            e = np.zeros((0, 8), np.uint32)
            return P.DualMesh(e, np.zeros(0, np.uint64), P.ExtractionStats()), P.ExtractionStats()
        d = P.extract_dual_mesh(dindex.index, cell_range=(lo, hi))
        return d, d.stats

    return partitioned_range(dindex.owned, run, group, device)


def partitioned_range(owned, extract_range, group=None, device=None):
    """partitioned() for an explicit owned range of local positions"""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    items, stats = extract_range(*owned)
    counts = allgather_counts(len(items), group, device)
    off = exclusive_offsets(counts)
    counters = allreduce_counters(stats, group, device)
    return PartitionedResult(items, int(off[rank]), int(off[-1]), counts, owned, stats,
                             counters)


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
    meta = meta.cpu().numpy()  # one host sync
    n = int(meta[0])
    geometry = meta[1:]
    if rank == src:  # broadcast straight from the index's own arrays (views)
        keys, scal = sorted_arrays(idx, dev)
        torch.cuda.synchronize(dev)  # the build ran on the library's stream
    else:
        keys = torch.empty(n, dtype=torch.int64, device=dev)
        scal = torch.empty(n, dtype=torch.float64, device=dev)
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
