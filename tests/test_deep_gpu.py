"""The deep configuration (SURVEY §8 "next": a hierarchy of >= 10 levels in
the style of the paper's 13-level landing gear): octrees
refined toward a landing-gear surface (synth.octree_sdf), shuffled into a
soup.  Their key spaces are far too sparse for a record per bucket, so the
index takes the hashed records; every output must equal the reference
library's bit for bit, and the forced directory must agree too."""
import numpy as np
import pytest

import oracles

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    R = oracles.reference()
    if R is None:
        pytest.skip("oracle/_ref not built")
    import paper_2004_08475_b200 as P
    from paper_2004_08475_b200 import synth
    return P, R, synth, torch


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("levels,root,lookup,expect", [
    (11, (1, 1, 1), None, "hash"),        # 34-bit keys, 2.2M cells: records would be 4 GB
    (10, (3, 2, 2), None, "hash"),
    (9, (3, 2, 2), "hash", "hash"),
    (9, (3, 2, 2), "directory", "directory"),
    (8, (2, 2, 2), "records", "records")])
def test_deep_octree_vs_reference(env, levels, root, lookup, expect):
    P, R, synth, torch = env
    cells, scal = synth.octree_sdf(root, levels, 0.9, device="cpu")
    cells, scal = cells.numpy(), scal.numpy()
    assert len(np.unique(cells[:, 3])) >= levels - 2  # a root cell may be refined away
    idx = P.build_index(cells, scal, lookup=lookup)
    assert idx.info.lookup == expect
    if expect == "hash":
        assert idx.info.max_probe < 64
    h = R.build(cells, scal)
    ds = R.dataset(h)
    assert (idx.cells == ds.cells).all() and (bits(idx.scalars) == bits(ds.scalars)).all()
    rd = R.extract_dual(h, 0)
    d = P.extract_dual_mesh(idx)
    assert d.corners.shape == rd["corners"].shape and (d.corners == rd["corners"]).all()
    ri = R.extract_iso(h, 0.0, 0)
    r = P.extract_isosurface(idx, P.IsoParams(iso=0.0))
    st = ri["stats"]
    assert [r.stats.duals_accepted, r.stats.duals_missing_corner, r.stats.duals_finer_corner,
            r.stats.duals_lower_key_corner] == [st["duals_accepted"], st["duals_missing_corner"],
                                                st["duals_finer_corner"],
                                                st["duals_lower_key_corner"]]
    assert r.fat.shape == ri["fat"].shape and (bits(r.fat) == bits(ri["fat"])).all()
    # the reference's own validator agrees the data is a proper octree
    rep = P.validate_dataset(idx)
    assert rep.ok()
    R.free(h)


def test_deep_queries_vs_reference(env):
    """snap / find_exact through the hashed records on a deep index"""
    P, R, synth, torch = env
    cells, scal = synth.octree_sdf((2, 2, 2), 9, 0.9, device="cpu")
    cells, scal = cells.numpy(), scal.numpy()
    idx = P.build_index(cells, scal, lookup="hash")
    assert idx.info.lookup == "hash"
    h = R.build(cells, scal)
    rng = np.random.default_rng(11)
    lo, hi = idx.bounds
    pts = np.stack([rng.integers(lo[a] - 5, hi[a] + 5, 4000) for a in range(3)], 1)
    hints = rng.integers(-1, 12, 4000).astype(np.int32)
    got = P.snap(idx, pts, hints)
    exp = np.array([R.snap(h, pts[i], int(hints[i])) for i in range(len(pts))])
    assert (got == exp).all()
    q = np.concatenate([cells[:3000], cells[:3000] + np.array([0, 0, 1 << 3, 0], np.int32)])
    got = P.find_exact(idx, q)
    exp = np.array([R.find_exact(h, q[i]) for i in range(len(q))])
    assert (got == exp).all()
    R.free(h)
