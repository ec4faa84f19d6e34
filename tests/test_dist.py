"""Multi-process (world_size 2 and 3, gloo, CPU) tests of the range-partition
plumbing in paper_2004_08475_b200/dist.py: rank 0 broadcasts the sorted index
arrays, every rank extracts its contiguous cell slice, counts are all-gathered
into global offsets, and the slices -- placed at those offsets -- reassemble
exactly the single-process output.  The oracle restatement stands in for the
GPU extractor (no GPU here); the GPU extractor itself is covered by the
range-partition test in test_gpu_parity.py."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "cases.npz")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _Stats:
    def __init__(self, c):
        (self.duals_accepted, self.duals_missing_corner, self.duals_finer_corner,
         self.duals_lower_key_corner) = [int(x) for x in c]


def worker(rank, world, port, case, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracles
        from paper_2004_08475_b200 import dist as D
        orc = oracles.restatement()
        z = np.load(GOLD)
        # rank 0 owns the (unsorted) input and sorts it; the sorted arrays are
        # broadcast, the other ranks adopt them presorted
        meta = torch.zeros(1, dtype=torch.int64)
        if rank == 0:
            h0 = orc.build(z[f"{case}/in_cells"], z[f"{case}/in_scalars"])
            ds = orc.dataset(h0)
            orc.free(h0)
            cells = torch.from_numpy(ds.cells.copy())
            scal = torch.from_numpy(ds.scalars.copy())
            meta[0] = len(cells)
        dist.broadcast(meta, 0)
        n = int(meta[0])
        if rank != 0:
            cells = torch.empty((n, 4), dtype=torch.int32)
            scal = torch.empty(n, dtype=torch.float64)
        dist.broadcast(cells, 0)
        dist.broadcast(scal, 0)
        h = orc.build(cells.numpy(), scal.numpy())
        iso = float(z[f"{case}/iso"])

        def run(lo, hi):
            r = orc.extract_iso(h, iso, lo, hi)
            return r["fat"], _Stats(r["counters"])

        res = D.partitioned(n, run)
        # gather the slices at their offsets on rank 0
        sizes = res.counts
        flat = torch.from_numpy(np.ascontiguousarray(res.fat).reshape(-1))
        pad = torch.zeros(max(sizes) * 9, dtype=torch.float64)
        pad[: flat.numel()] = flat
        bufs = [torch.zeros_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad)
        if rank == 0:
            full = np.zeros((res.total, 9))
            off = D.exclusive_offsets(sizes)
            for r in range(world):
                full[off[r]: off[r + 1]] = bufs[r][: sizes[r] * 9].numpy().reshape(-1, 9)
            q.put(("ok", full, res.counters, res.total, sizes))
        orc.free(h)
    except Exception as e:  # surface failures to the parent
        q.put(("err", repr(e), None, None, None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, "slots_l4_s3"), (3, "octree_sphere"),
                                        (2, "acceptance_34")])
def test_partitioned_iso_reassembles_single_output(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    status, full, counters, total, sizes = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
    assert status == "ok", full
    z = np.load(GOLD)
    ref = z[f"{case}/fat"]
    assert total == len(ref) and sum(sizes) == total
    assert (full.view(np.uint64) == ref.view(np.uint64)).all()
    assert list(counters) == [int(x) for x in z[f"{case}/counters"]]


def test_cell_range_covers_exactly():
    from paper_2004_08475_b200 import dist as D
    for n in (0, 1, 7, 100, 12345):
        for world in (1, 2, 3, 8):
            ranges = [D.cell_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(ranges[r][1] == ranges[r + 1][0] for r in range(world - 1))
    assert list(D.exclusive_offsets([3, 0, 5])) == [0, 3, 3, 8]


# --------------------------------------------------------------------------
# distributed build (dist.build_distributed): the exchange plan over gloo.
# Keys are packed here in the library's layout (major field i, then j, k,
# level; geometry word 15 carries the layout) from a golden case's cells.

def _packed(case):
    z = np.load(GOLD)
    cells = z[f"{case}/in_cells"].astype(np.int64)
    mn = cells[:, :3].min(0)
    levels = sorted(set(cells[:, 3].tolist()))
    shift, coarsest = levels[0], levels[-1]
    bits = [int((cells[:, a].max() - mn[a]) >> shift).bit_length() for a in range(3)]
    lbits = int(coarsest - shift).bit_length()
    sh2 = lbits
    sh1 = sh2 + bits[2]
    sh0 = sh1 + bits[1]
    keys = ((cells[:, 3] - shift) | (((cells[:, 0] - mn[0]) >> shift) << sh0) |
            (((cells[:, 1] - mn[1]) >> shift) << sh1) | (((cells[:, 2] - mn[2]) >> shift) << sh2))
    total = sh0 + bits[0]
    major = sh0 if bits[0] else (sh1 if bits[1] else (sh2 if bits[2] else lbits))
    g = np.zeros(16, np.int64)
    g[15] = major | (shift << 8) | (coarsest << 16) | (total << 24)
    return keys.astype(np.int64), z[f"{case}/in_scalars"], g


def exchange_worker(rank, world, port, case, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2004_08475_b200 import dist as D
        keys, scal, g = _packed(case)
        n = len(keys)
        a, b = n * rank // world, n * (rank + 1) // world
        k = torch.from_numpy(keys[a:b])
        s = torch.from_numpy(np.ascontiguousarray(scal[a:b]))
        order = torch.argsort(k)
        k, s = k[order].contiguous(), s[order].contiguous()
        pos = torch.linspace(0, len(k) - 1, 32).round().long()
        smp = k[pos]
        got = [torch.empty_like(smp) for _ in range(world)]
        dist.all_gather(got, smp)
        bounds = D.choose_splitters(torch.cat(got), world)
        lo, hi = D.halo_ranges(bounds, g)
        rk, rs = D.exchange_runs(k, s, lo, hi)
        below, own = D.owned_split(rk, bounds, rank)
        owns = D.allgather_counts(own)
        id_base = sum(owns[:rank]) - below
        # what this rank must hold: every key in [lo, hi), each once
        full = np.sort(keys)
        want = full[(full >= lo[rank]) & (full < hi[rank])]
        mine = np.sort(rk.numpy())
        ok = len(mine) == len(want) and (mine == want).all()
        # scalars travel with their keys
        kv = dict(zip(keys.tolist(), scal.tolist()))
        ok = ok and all(kv[int(x)] == float(y) for x, y in zip(rk.numpy(), rs.numpy()))
        # the owned ranges tile the key space; local sorted position + id_base
        # is the key's global CellId
        ok = ok and sum(owns) == n
        gid = np.searchsorted(full, mine)
        ok = ok and (gid == id_base + np.arange(len(mine))).all()
        q.put(("ok" if ok else "mismatch", rank))
    except Exception as e:
        q.put(("err", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, "slots_l4_s3"), (3, "octree_sphere"),
                                        (3, "blocks_jump2")])
def test_distributed_exchange_plan(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=exchange_worker, args=(r, world, port, case, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[0] == "ok" for r in res), res


def test_halo_ranges_cover_owned():
    from paper_2004_08475_b200 import dist as D
    _, _, g = _packed("blocks_jump2")
    msh, finest, coarsest, bits = D.geometry_layout(g)
    bounds = [0, 1000, 5000, 1 << 63]
    lo, hi = D.halo_ranges(bounds, g)
    for q in range(3):
        a, b = bounds[q], min(bounds[q + 1], 1 << bits)
        assert lo[q] <= a and hi[q] >= b
        assert lo[q] % (1 << msh) == 0
