"""Two-word (> 64-bit) keys (csrc/wide.cuh, wide.cu): datasets whose extent
needs more than 64 key bits build and extract exactly like the reference
(proj/include/amriso/core.hpp:82-88 accepts any int32 anchor on levels
0..30; proj/src/locator.cpp:26-50).  Golden datasets are placed twice, far
apart, so the key spans ~3 x 31 bits; every output -- sorted arrays, duals,
task ids, counters, FP64 soup bits, snap / find_exact / try_build_dual /
validate -- is compared with the reference library bit for bit."""
import os

import numpy as np
import pytest

import oracles

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _cases():
    z = np.load(os.path.join(HERE, "golden", "cases.npz"))
    names = sorted({k.split("/")[0] for k in z.files})
    return {n: {k.split("/")[1]: z[k] for k in z.files if k.startswith(n + "/")} for n in names}


CASES = _cases()


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    R = oracles.reference()
    if R is None:
        pytest.skip("oracle/_ref not built")
    import paper_2004_08475_b200 as P
    return P, R


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def far_apart(cells, scal, seed):
    """two copies of a dataset, the second moved by ~2^30 on every axis
    (aligned to its coarsest level), shuffled together"""
    top = int(cells[:, 3].max())
    off = np.array([(1 << 30) - (1 << top), (1 << 30) - (2 << top), (1 << 30) - (3 << top), 0],
                   np.int64)
    c2 = (cells.astype(np.int64) + off)
    assert (c2[:, :3] < 2**31).all()
    c = np.concatenate([cells.astype(np.int64), c2]).astype(np.int32)
    s = np.concatenate([scal, -scal])
    perm = np.random.default_rng(seed).permutation(len(c))
    return c[perm], s[perm]


@pytest.mark.parametrize("name", ["slots_l4_s3", "octree_sphere", "blocks_jump2",
                                  "acceptance_1"])
def test_wide_vs_reference(env, name):
    P, R = env
    cc = CASES[name]
    cells, scal = far_apart(cc["in_cells"], cc["in_scalars"], 5)
    iso = float(cc["iso"])
    idx = P.build_index(cells, scal)
    assert idx.info.key_bits > 64 and idx.info.lookup == "wide"
    h = R.build(cells, scal)
    ds = R.dataset(h)
    assert (idx.cells == ds.cells).all() and (bits(idx.scalars) == bits(ds.scalars)).all()
    assert idx.levels == [int(x) for x in ds.levels]
    rd = R.extract_dual(h, 0)
    d = P.extract_dual_mesh(idx)
    assert d.corners.shape == rd["corners"].shape and (d.corners == rd["corners"]).all()
    ri = R.extract_iso(h, iso, 0)
    r = P.extract_isosurface(idx, P.IsoParams(iso=iso))
    st = ri["stats"]
    assert [r.stats.duals_accepted, r.stats.duals_missing_corner, r.stats.duals_finer_corner,
            r.stats.duals_lower_key_corner] == [st["duals_accepted"], st["duals_missing_corner"],
                                                st["duals_finer_corner"],
                                                st["duals_lower_key_corner"]]
    assert r.fat.shape == ri["fat"].shape and (bits(r.fat) == bits(ri["fat"])).all()
    # the copy far away is the same mesh shifted: twice the duals
    assert len(d) == 2 * len(cc["dual_corners"])
    # device and pinned outputs, f32 soup
    import torch
    out = torch.empty((len(r.fat), 9), dtype=torch.float64, device="cuda")
    r2 = P.extract_isosurface(idx, P.IsoParams(iso=iso), out=out)
    assert (bits(r2.fat.cpu().numpy()) == bits(ri["fat"])).all()
    pin = torch.empty((len(r.fat), 9), dtype=torch.float64, pin_memory=True)
    r3 = P.extract_isosurface(idx, P.IsoParams(iso=iso), out=pin)
    assert (bits(r3.fat.numpy()) == bits(ri["fat"])).all()
    rf = P.extract_isosurface(idx, P.IsoParams(iso=iso, f32=True))
    ref = ri["fat"]
    rel = np.abs(rf.fat.astype(np.float64) - ref) / np.maximum(np.abs(ref), 1.0)
    assert len(ref) == 0 or rel.max() <= 1e-5
    R.free(h)


def test_wide_queries_vs_reference(env):
    P, R = env
    cc = CASES["slots_l4_s3"]
    cells, scal = far_apart(cc["in_cells"], cc["in_scalars"], 7)
    idx = P.build_index(cells, scal)
    h = R.build(cells, scal)
    ds = R.dataset(h)
    rng = np.random.default_rng(9)
    lo, hi = idx.bounds
    # points near both copies and in the empty space between them
    base = ds.cells[rng.integers(0, len(ds), 3000), :3].astype(np.int64)
    pts = np.concatenate([base + rng.integers(-40, 40, (3000, 3)),
                          rng.integers(lo, np.array(hi) + 1, (1000, 3))])
    hints = rng.integers(-1, 31, len(pts)).astype(np.int32)
    got = P.snap(idx, pts, hints)
    exp = np.array([R.snap(h, pts[i], int(hints[i])) for i in range(len(pts))])
    assert (got == exp).all()
    q = np.concatenate([ds.cells[:2000], ds.cells[:2000] + np.array([1, 0, 0, 0], np.int32),
                        ds.cells[:2000] + np.array([0, 0, 0, 1], np.int32)])
    got = P.find_exact(idx, q)
    exp = np.array([R.find_exact(h, q[i]) for i in range(len(q))])
    assert (got == exp).all()
    n = len(ds)
    tasks = np.arange(0, 8 * n, 3, dtype=np.uint64)
    rej, cor = P.try_build_duals(idx, tasks)
    base_, lev = P.dual_bases(idx, tasks)
    for t in range(0, len(tasks), 11):
        r, corners = R.try_build_dual(h, base_[t], int(lev[t]), int(tasks[t] >> 3))
        assert r == rej[t]
        if r == 0:
            assert (corners == cor[t]).all()
    R.free(h)


def test_wide_validate_and_duplicates(env):
    """duplicates and overlaps in a wide index: validate pairs and the
    duplicate-key lookups (first of a run, like lower_bound)"""
    P, R = env
    cc = CASES["octree_sphere"]
    cells, scal = far_apart(cc["in_cells"], cc["in_scalars"], 3)
    extra = np.array([cells[0], cells[5], [cells[9][0] & ~7, cells[9][1] & ~7, cells[9][2] & ~7,
                                           3]], np.int32)
    cells = np.concatenate([cells, extra])
    scal = np.concatenate([scal, [1.0, 2.0, 3.0]])
    idx = P.build_index(cells, scal)
    assert idx.info.duplicate_keys == 2
    h = R.build(cells, scal)
    rep = P.validate_dataset(idx)
    dup, ovl = R.validate_pairs(h)
    assert (rep.duplicates == dup).all() and (rep.overlaps == ovl).all()
    d = P.extract_dual_mesh(idx)
    rd = R.extract_dual(h, 0)
    assert (d.corners == rd["corners"]).all()
    R.free(h)
