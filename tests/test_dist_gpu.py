"""The distributed build (dist.build_distributed) on one GPU: every rank's
steps -- bounds, slice sort, sampled splitters, halo ranges, the exchange,
partition index with its global id base, owned-range extraction -- run in
turn in one process, with the all-to-all done by slicing.  Concatenated in
rank order the partitions' outputs must equal the single-GPU extraction
bit for bit (dual corners + task ids, the FP64 soup, the reject counters).
The collectives themselves are covered over gloo in tests/test_dist.py."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2004_08475_b200 as P
    from paper_2004_08475_b200 import dist as D
    return P, D, torch


def emulate(P, D, torch, cells, scal, world, samples=64, lookup=None):
    dev = torch.device("cuda", 0)
    n = len(cells)
    cut = [n * r // world for r in range(world + 1)]
    sl = [(cells[cut[r]:cut[r + 1]], scal[cut[r]:cut[r + 1]]) for r in range(world)]
    allb = np.stack([np.append(P.cell_bounds(c), len(c)) for c, _ in sl])
    g = D.global_geometry(allb[:, :10], allb[:, 10])
    arrays, parts_sorted = [], []
    for c, s in sl:
        part = P.sort_part(c, s, g)
        gg = part.geometry()
        arrays.append(D.sorted_arrays(part, dev))  # zero-copy views: keep `part` open
        parts_sorted.append(part)
    gg[10] = n
    smp = []
    for k, _ in arrays:
        pos = torch.linspace(0, len(k) - 1, samples, device=dev).round().long()
        smp.append(k[pos])
    bounds = D.choose_splitters(torch.cat(smp), world)
    lo, hi = D.halo_ranges(bounds, gg)
    plans = [D.send_plan(k, lo, hi) for k, _ in arrays]
    recv = []
    for r in range(world):
        ks = [arrays[q][0][plans[q][0][r]:plans[q][0][r] + plans[q][1][r]] for q in range(world)]
        ss = [arrays[q][1][plans[q][0][r]:plans[q][0][r] + plans[q][1][r]] for q in range(world)]
        recv.append((torch.cat(ks), torch.cat(ss)))
    torch.cuda.synchronize()
    del arrays
    for part in parts_sorted:
        part.close()
    split = [D.owned_split(rk, bounds, r) for r, (rk, _) in enumerate(recv)]
    owns = [o for _, o in split]
    assert sum(owns) == n
    parts = []
    for r, (rk, rs) in enumerate(recv):
        below, own = split[r]
        g2 = gg.copy()
        g2[12], g2[13], g2[14] = sum(owns[:r]) - below, lo[r], hi[r]
        idx = P.index_from_keys(rk.data_ptr(), rs.data_ptr(), len(rk), g2,
                                lookup=lookup) if own else None
        if idx is not None and lookup:
            assert idx.info.lookup == lookup
        parts.append((idx, (below, below + own)))
    return parts


def check(P, D, torch, cells, scal, iso, world, lookup=None):
    ref = P.build_index(cells, scal)
    d_ref = P.extract_dual_mesh(ref)
    r_ref = P.extract_isosurface(ref, P.IsoParams(iso=iso))
    parts = emulate(P, D, torch, cells, scal, world, lookup=lookup)
    corners, tasks, fats, counters = [], [], [], np.zeros(4, np.int64)
    for idx, (lo, hi) in parts:
        if idx is None:
            continue
        d = P.extract_dual_mesh(idx, cell_range=(lo, hi))
        corners.append(d.corners)
        tasks.append(d.tasks)
        r = P.extract_isosurface(idx, P.IsoParams(iso=iso), cell_range=(lo, hi))
        fats.append(r.fat)
        s = r.stats
        counters += [s.duals_accepted, s.duals_missing_corner, s.duals_finer_corner,
                     s.duals_lower_key_corner]
        idx.close()
    assert (np.concatenate(corners) == d_ref.corners).all()
    assert (np.concatenate(tasks) == d_ref.tasks).all()
    fat = np.concatenate(fats)
    assert fat.shape == r_ref.fat.shape
    assert (fat.view(np.uint64) == r_ref.fat.view(np.uint64)).all()
    s = r_ref.stats
    assert list(counters) == [s.duals_accepted, s.duals_missing_corner, s.duals_finer_corner,
                              s.duals_lower_key_corner]


def _cases():
    z = np.load(os.path.join(HERE, "golden", "cases.npz"))
    names = sorted({k.split("/")[0] for k in z.files})
    return {n: {k.split("/")[1]: z[k] for k in z.files if k.startswith(n + "/")} for n in names}


CASES = _cases()


@pytest.mark.parametrize("lookup", [None, "hash"])
@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("name", ["slots_l4_s3", "octree_sphere", "blocks_jump2", "acceptance_1"])
def test_partitions_reproduce_single_gpu(env, name, world, lookup):
    P, D, torch = env
    c = CASES[name]
    check(P, D, torch, c["in_cells"], c["in_scalars"], float(c["iso"]), world, lookup)


def test_partition_refuses_queries_and_halo_ranges(env):
    """a partition holds one key range plus its halo: point queries and
    extraction ranges reaching into the halo are refused (their answers
    would need other ranks' cells), the owned range is accepted"""
    P, D, torch = env
    from paper_2004_08475_b200 import synth
    ds = synth.bricks([16, 8, 8], seed=3, shuffle=True, holes=synth.body_holes([16, 8, 8]))
    cells, scal = ds.cells.cpu().numpy(), ds.scalars.cpu().numpy()
    c = {"cells": cells}
    parts = emulate(P, D, torch, cells, scal, 4)
    checked = 0
    for idx, (lo, hi) in parts:
        if idx is None:
            continue
        with pytest.raises(ValueError, match="partition"):
            P.find_exact(idx, c["cells"][:4])
        with pytest.raises(ValueError, match="partition"):
            P.snap(idx, c["cells"][:4, :3].astype(np.int64))
        with pytest.raises(ValueError, match="partition"):
            P.validate_dataset(idx)
        P.extract_dual_mesh(idx, cell_range=(lo, hi))
        if idx.geometry()[13] > 0:  # the key range (owned + halo) starts above key 0
            with pytest.raises(ValueError, match="interior"):
                P.extract_dual_mesh(idx, cell_range=(0, hi))
            checked += 1
        idx.close()
    assert checked >= 1


@pytest.mark.parametrize("world", [2, 8])
def test_partitions_bricks(env, world):
    """the block-structured generator (level jumps up to 3, holes), shuffled"""
    P, D, torch = env
    from paper_2004_08475_b200 import synth
    b3 = [16, 8, 8]
    ds = synth.bricks(b3, seed=3, shuffle=True, holes=synth.body_holes(b3))
    cells = ds.cells.cpu().numpy() if hasattr(ds.cells, "cpu") else np.asarray(ds.cells)
    scal = ds.scalars.cpu().numpy() if hasattr(ds.scalars, "cpu") else np.asarray(ds.scalars)
    check(P, D, torch, cells, scal, synth.C4_ISO, world)
