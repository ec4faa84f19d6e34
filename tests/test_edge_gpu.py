"""Edge cases of the GPU path against the C restatement: one cell, a 2x2x2
block, a single column, a constant axis, a range that covers nothing, and an
iso value no scalar crosses."""
import numpy as np
import pytest

from conftest import LOOKUPS, LookupProxy

import oracles

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=LOOKUPS)
def P(request):
    """the package, once per lookup structure (conftest.LookupProxy)"""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2004_08475_b200 as P
    return LookupProxy(P, request.param)


def same(P, cells, scal, iso):
    cells = np.ascontiguousarray(np.asarray(cells, np.int32).reshape(-1, 4))
    scal = np.ascontiguousarray(np.asarray(scal, np.float64))
    idx = P.build_index(cells, scal)
    orc = oracles.restatement()
    h = orc.build(cells, scal)
    d = P.extract_dual_mesh(idx)
    od = orc.extract_dual(h)
    assert d.corners.shape == od["corners"].shape and (d.corners == od["corners"]).all()
    r = P.extract_isosurface(idx, P.IsoParams(iso=iso))
    oi = orc.extract_iso(h, iso)
    assert r.fat.shape == oi["fat"].shape
    assert (r.fat.view(np.uint64) == oi["fat"].view(np.uint64)).all()
    assert [r.stats.duals_accepted, r.stats.duals_missing_corner, r.stats.duals_finer_corner,
            r.stats.duals_lower_key_corner] == [int(x) for x in oi["counters"]]
    orc.free(h)
    return idx, r


def test_one_cell(P):
    idx, r = same(P, [[0, 0, 0, 0]], [1.0], 0.5)
    assert len(r.fat) == 0 and r.stats.duals_missing_corner == 8


def test_block_2x2x2(P):
    c = [[i, j, k, 0] for k in range(2) for j in range(2) for i in range(2)]
    s = [float(i + 2 * j + 4 * k) for (i, j, k, _) in c]
    idx, r = same(P, c, s, 3.5)
    assert r.stats.duals_accepted == 1 and len(r.fat) > 0


def test_single_column_and_constant_axis(P):
    c = [[0, 0, k, 1] for k in range(0, 64, 2)]
    same(P, c, np.linspace(-1, 1, len(c)), 0.0)
    c = [[i, 4, k, 0] for k in range(6) for i in range(5)]  # y constant
    same(P, c, np.sin(np.arange(len(c))), 0.1)


def test_negative_anchors_and_levels(P):
    rng = np.random.default_rng(3)
    c = []
    for k in range(-4, 4):
        for j in range(-4, 4):
            for i in range(-8, 0):
                c.append([i, j, k, 0])
    for k in range(-4, 4, 2):
        for j in range(-4, 4, 2):
            for i in range(0, 8, 2):
                c.append([i, j, k, 1])
    c = np.array(c)
    same(P, c[rng.permutation(len(c))], rng.normal(size=len(c)), 0.0)


def test_empty_range_and_no_crossing(P):
    c = [[i, j, k, 0] for k in range(4) for j in range(4) for i in range(4)]
    idx = P.build_index(np.array(c, np.int32), np.ones(len(c)))
    r = P.extract_isosurface(idx, P.IsoParams(iso=5.0))
    assert len(r.fat) == 0 and r.stats.duals_accepted == 27
    d = P.extract_dual_mesh(idx, cell_range=(10, 10))
    assert len(d.corners) == 0


def test_level30_cells_span_the_int32_range(P):
    """Coarsest legal level (locator.cpp:38-41: level <= 30): a 4x4x4 block of
    level-30 cells whose anchors cover [-2^31, 2^31), one of them refined into
    eight level-29 cells.  Stencil points and dual bases leave the int32 range
    here, which snap rejects by its range guard (locator.cpp:107-115)."""
    W = 1 << 30
    c = [[i * W, j * W, k * W, 30] for k in range(-2, 2) for j in range(-2, 2)
         for i in range(-2, 2) if (i, j, k) != (0, 0, 0)]
    H = 1 << 29
    c += [[i * H, j * H, k * H, 29] for k in range(2) for j in range(2) for i in range(2)]
    c = np.array(c, np.int64)
    rng = np.random.default_rng(30)
    scal = rng.normal(size=len(c))
    idx, r = same(P, c[rng.permutation(len(c))], scal, 0.0)
    assert r.stats.duals_accepted > 0


def test_key_wider_than_64_bits(P):
    """Fine cells spread across the whole int32 range need a packed key of
    more than 64 bits (3 x 32 coordinate bits + the level field): the index
    takes two-word keys (csrc/wide.cuh) and every output equals the
    restatement bit for bit (locator.cpp:26-50 accepts these inputs)."""
    lim = (1 << 31) - 2
    c = np.array([[-lim - 1, -lim - 1, -lim - 1, 0], [lim, lim, lim, 0], [0, 0, 0, 5],
                  [32, 0, 0, 5], [0, 32, 0, 5], [32, 32, 0, 5], [0, 0, 32, 5], [32, 0, 32, 5],
                  [0, 32, 32, 5], [32, 32, 32, 5], [lim - 1, lim, lim, 0]], np.int32)
    rng = np.random.default_rng(64)
    idx, r = same(P, c[rng.permutation(len(c))], rng.normal(size=len(c)), 0.0)
    assert idx.info.key_bits > 64 and idx.info.lookup == "wide"
    assert r.stats.duals_accepted >= 1
