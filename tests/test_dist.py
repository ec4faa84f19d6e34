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
