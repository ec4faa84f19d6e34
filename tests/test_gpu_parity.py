"""GPU parity: the CUDA path (through the C ABI) against the reference.

Every comparison is bit-exact (integer ids, counters, FP64 vertex bits) --
the north star's bar for duals ("bit-exact after canonical sorting") is met
without the canonical sort because our output order IS the reference's
candidate order; the f32 soup is checked at the 1e-5 relative tolerance.

Sources of truth: the committed golden vectors (tests/golden/, produced by
the reference itself), the C restatement (oracle/liboracle.so) and, where it
was built, the reference library (oracle/_ref)."""
import json
import os

import numpy as np
import pytest

import oracles
from conftest import LOOKUPS, LookupProxy

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def _cases():
    z = np.load(os.path.join(GOLD, "cases.npz"))
    names = sorted({k.split("/")[0] for k in z.files})
    return {n: {k.split("/")[1]: z[k] for k in z.files if k.startswith(n + "/")} for n in names}


CASES = _cases()
KNOWN = json.load(open(os.path.join(GOLD, "known_answers.json")))


@pytest.fixture(scope="module", params=LOOKUPS)
def P(request):
    """the package, once per lookup structure (conftest.LookupProxy)"""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2004_08475_b200 as P
    return LookupProxy(P, request.param)


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def check_against(P, idx, cells, scalars, levels, dual_corners, dual_tasks, counters, fat, iso):
    assert (idx.cells == cells).all()
    assert (bits(idx.scalars) == bits(scalars)).all()
    assert idx.levels == [int(x) for x in levels]
    d = P.extract_dual_mesh(idx)
    assert d.corners.shape == dual_corners.shape
    assert (d.corners == dual_corners).all()
    if dual_tasks is not None:
        assert (d.tasks == dual_tasks).all()
    r = P.extract_isosurface(idx, P.IsoParams(iso=iso))
    s = r.stats
    got = [s.duals_accepted, s.duals_missing_corner, s.duals_finer_corner,
           s.duals_lower_key_corner]
    assert got == [int(x) for x in counters]
    assert s.duals_accepted == len(dual_corners)
    assert s.pass1_triangle_count == s.fat_triangle_count == len(fat)
    assert r.fat.shape == fat.shape
    assert (bits(r.fat) == bits(fat)).all()
    return r


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_case(P, name):
    c = CASES[name]
    idx = P.build_index(c["in_cells"], c["in_scalars"])
    check_against(P, idx, c["cells"], c["scalars"], c["levels"], c["dual_corners"],
                  c["dual_tasks"], c["counters"], c["fat"], float(c["iso"]))
    lo, hi = idx.bounds
    assert list(lo) == list(c["bounds"][:3]) and list(hi) == list(c["bounds"][3:])


@pytest.mark.parametrize("name", sorted(CASES))
def test_golden_case_presorted(P, name):
    """already-sorted input skips the radix sort; results identical"""
    c = CASES[name]
    idx = P.build_index(c["cells"], c["scalars"], presorted=True)
    check_against(P, idx, c["cells"], c["scalars"], c["levels"], c["dual_corners"],
                  c["dual_tasks"], c["counters"], c["fat"], float(c["iso"]))


def test_f32_soup_within_tolerance(P):
    c = CASES["slots_l4_s3"]
    idx = P.build_index(c["in_cells"], c["in_scalars"])
    r = P.extract_isosurface(idx, P.IsoParams(iso=float(c["iso"]), f32=True))
    assert r.fat.dtype == np.float32 and r.fat.shape == c["fat"].shape
    ref = c["fat"]
    rel = np.abs(r.fat.astype(np.float64) - ref) / np.maximum(np.abs(ref), 1.0)
    assert rel.max() <= 1e-5


def test_device_output_buffers(P):
    import torch
    c = CASES["octree_sphere"]
    idx = P.build_index(torch.from_numpy(c["in_cells"]).cuda(),
                        torch.from_numpy(c["in_scalars"]).cuda())
    n = len(c["dual_corners"])
    corners = torch.empty((n, 8), dtype=torch.int32, device="cuda")
    tasks = torch.empty(n, dtype=torch.int64, device="cuda")
    d = P.extract_dual_mesh(idx, out=(corners, tasks))
    assert (d.corners.cpu().numpy().view(np.uint32) == c["dual_corners"]).all()
    fat = torch.empty((len(c["fat"]), 9), dtype=torch.float64, device="cuda")
    r = P.extract_isosurface(idx, P.IsoParams(iso=0.0), out=fat)
    assert (bits(r.fat.cpu().numpy()) == bits(c["fat"])).all()
    # too small a device buffer: capacity error carrying the needed count
    small = torch.empty((1, 9), dtype=torch.float64, device="cuda")
    with pytest.raises(P.CapacityError) as e:
        P.extract_isosurface(idx, P.IsoParams(iso=0.0), out=small)
    assert e.value.count == len(c["fat"])


def test_range_partition_concatenates(P):
    """per-range extraction in rank order == full extraction (the multi-GPU
    partition contract, pipeline.cpp:40-57 candidate order)"""
    c = CASES["slots_l4_s3"]
    idx = P.build_index(c["in_cells"], c["in_scalars"])
    n = len(idx)
    for parts in (2, 3, 8):
        cuts = [n * r // parts for r in range(parts + 1)]
        duals = [P.extract_dual_mesh(idx, cell_range=(cuts[r], cuts[r + 1])).corners
                 for r in range(parts)]
        assert (np.concatenate(duals) == c["dual_corners"]).all()
        fats = [P.extract_isosurface(idx, float(c["iso"]), cell_range=(cuts[r], cuts[r + 1])).fat
                for r in range(parts)]
        assert (bits(np.concatenate(fats)) == bits(c["fat"])).all()


def test_find_exact_and_snap(P, orc):
    rng = np.random.default_rng(7)
    for name in ("slots_s11", "slots_l4_s3", "octree_sphere", "blocks_jump2"):
        c = CASES[name]
        idx = P.build_index(c["in_cells"], c["in_scalars"])
        ho = orc.build(c["cells"], c["scalars"])
        lo, hi = c["bounds"][:3], c["bounds"][3:]
        pts = np.stack([rng.integers(lo[a] - 3, hi[a] + 3, 3000) for a in range(3)], 1)
        hints = rng.integers(-1, 31, 3000).astype(np.int32)
        got = P.snap(idx, pts, hints)
        exp = [orc.snap(ho, pts[i], int(hints[i])) for i in range(len(pts))]
        assert (got == np.array(exp)).all()
        got0 = P.snap(idx, pts, -1)
        exp0 = [orc.snap(ho, pts[i], -1) for i in range(len(pts))]
        assert (got0 == np.array(exp0)).all()
        # find_exact: stored keys hit themselves, perturbed keys mostly miss
        q = np.concatenate([c["cells"], c["cells"] + np.array([1, 0, 0, 0], np.int32),
                            c["cells"] + np.array([0, 0, 0, 1], np.int32)])
        got = P.find_exact(idx, q)
        exp = [orc.find_exact(ho, q[i]) for i in range(len(q))]
        assert (got == np.array(exp)).all()
        orc.free(ho)


def test_try_build_duals(P, orc):
    c = CASES["slots_l4_s3"]
    idx = P.build_index(c["in_cells"], c["in_scalars"])
    ho = orc.build(c["cells"], c["scalars"])
    n = len(c["cells"])
    tasks = np.arange(8 * n, dtype=np.uint64)
    rej, cor = P.try_build_duals(idx, tasks)
    base, lev = P.dual_bases(idx, tasks)
    for t in range(0, 8 * n, 7):
        r, corners = orc.try_build_dual(ho, base[t], int(lev[t]), int(t >> 3))
        assert r == rej[t]
        if r == 0:
            assert (corners == cor[t]).all()
    assert np.bincount(rej, minlength=4).tolist() == [int(x) for x in c["counters"]]
    orc.free(ho)


def test_int32_boundary(P):
    """snap stays exact at the 32-bit anchor boundary (test_locator.cpp:137-153)"""
    hi, lo = 2**31 - 1, -2**31
    idx = P.build_index(np.array([[hi, 0, 0, 0], [lo, 0, 0, 0]], np.int32), np.array([1.0, 2.0]))
    top = P.snap(idx, [[hi, 0, 0]])[0]
    assert top >= 0 and idx.cells[top][0] == hi
    assert P.snap(idx, [[hi + 1, 0, 0]])[0] == -1
    bot = P.snap(idx, [[lo, 0, 0]])[0]
    assert bot >= 0 and idx.cells[bot][0] == lo
    assert P.snap(idx, [[lo - 1, 0, 0]])[0] == -1
    d = P.extract_dual_mesh(idx)
    assert len(d) == 0


def test_load_errors_name_the_record(P):
    with pytest.raises(P.LoadError, match="record 2"):
        P.build_index(np.array([[0, 0, 0, 0], [0, 0, 0, 0], [0, 0, 0, 31]], np.int32),
                      np.zeros(3))
    with pytest.raises(P.LoadError, match="record 1: anchor .* not a multiple"):
        P.build_index(np.array([[0, 0, 0, 1], [2, 2, 1, 1]], np.int32), np.zeros(2))
    with pytest.raises(P.LoadError, match="record 0: level -1"):
        P.build_index(np.array([[0, 0, 0, -1]], np.int32), np.zeros(1))


def test_duplicates_follow_lower_bound(P, orc):
    """duplicate keys (invalid data the library still accepts): ties keep
    input order and lookups return the first duplicate, like lower_bound"""
    cells = np.array([[0, 0, 0, 0], [1, 0, 0, 0], [0, 0, 0, 0], [0, 1, 0, 0], [1, 1, 0, 0]],
                     np.int32)
    sc = np.array([1.0, 2.0, 3.0, 4.0, 5.0])
    idx = P.build_index(cells, sc)
    ho = orc.build(cells, sc)
    ds = orc.dataset(ho)
    assert (idx.cells == ds.cells).all() and (bits(idx.scalars) == bits(ds.scalars)).all()
    d = P.extract_dual_mesh(idx)
    od = orc.extract_dual(ho)
    assert (d.corners == od["corners"]).all()
    r = P.extract_isosurface(idx, 2.5)
    assert [r.stats.duals_accepted, r.stats.duals_missing_corner, r.stats.duals_finer_corner,
            r.stats.duals_lower_key_corner] == od["counters"].tolist()
    orc.free(ho)


def test_acceptance_pool_vs_reference(P, ref):
    """the 102 acceptance datasets, each bit-exact against the reference;
    totals as acceptance.cpp reports them"""
    tot_d = tot_t = 0
    for n in range(102):
        h, iso = ref.acceptance_fixture(n)
        ds = ref.dataset(h)
        perm = np.random.default_rng(n).permutation(len(ds))
        idx = P.build_index(ds.cells[perm], ds.scalars[perm])
        rd = ref.extract_dual(h, 0)
        ri = ref.extract_iso(h, iso, 0)
        st = ri["stats"]
        check_against(P, idx, ds.cells, ds.scalars, ds.levels, rd["corners"], None,
                      [st["duals_accepted"], st["duals_missing_corner"], st["duals_finer_corner"],
                       st["duals_lower_key_corner"]], ri["fat"], iso)
        tot_d += len(rd["corners"])
        tot_t += len(ri["fat"])
        ref.free(h)
    assert (tot_d, tot_t) == (74877, 116719)


@pytest.mark.parametrize("seed", [1, 5, 9])
def test_exhaustive_duals_level_jumps_to_4(P, ref, seed):
    """dual set == exhaustive enumeration on slot data with 0..4 level jumps
    (acceptance.cpp:182-203 generalised)"""
    h = ref.gen_slots(seed, 3, 4, 0.15)
    ds = ref.dataset(h)
    idx = P.build_index(ds.cells, ds.scalars)
    keys = ref.exhaustive_duals(h)
    d = P.extract_dual_mesh(idx)
    mine = np.sort(d.corners, axis=1)
    mine = mine[np.lexsort(mine.T[::-1])]
    assert mine.shape == keys.shape and (mine == keys).all()
    ref.free(h)


@pytest.mark.parametrize("which", ["octree7", "slots_l4_s6_n6", "c1_octree6"])
def test_larger_known_answers(P, ref, which):
    gens = {"octree7": lambda: ref.gen_octree(7, "sphere", [50, 55, 60, 40.0], 3.2),
            "slots_l4_s6_n6": lambda: ref.gen_slots(6, 6, 4, 0.15),
            "c1_octree6": lambda: ref.gen_octree(6, "sphere", [25, 27.5, 30, 20.0], 3.2)}
    iso = 0.1 if which.startswith("slots") else 0.0
    h = gens[which]()
    ds = ref.dataset(h)
    perm = np.random.default_rng(3).permutation(len(ds))
    idx = P.build_index(ds.cells[perm], ds.scalars[perm])
    rd = ref.extract_dual(h, 0)
    ri = ref.extract_iso(h, iso, 0)
    st = ri["stats"]
    check_against(P, idx, ds.cells, ds.scalars, ds.levels, rd["corners"], None,
                  [st["duals_accepted"], st["duals_missing_corner"], st["duals_finer_corner"],
                   st["duals_lower_key_corner"]], ri["fat"], iso)
    k = KNOWN[which]
    assert st["fat_triangle_count"] == k["fat_triangle_count"]
    ref.free(h)


def test_dual_cells_records(P, ref):
    """amrx_extract_dual_cells: the reference's DualCell records (corners,
    base = dual_base_of(owner, delta), level, owner) built on the device"""
    c = CASES["slots_l4_s3"]
    idx = P.build_index(c["in_cells"], c["in_scalars"])
    recs = P.extract_dual_cells(idx)
    h = ref.build(c["in_cells"], c["in_scalars"])
    rd = ref.extract_dual(h, 0)
    assert (recs["corners"] == rd["corners"]).all()
    assert (recs["owner"] == rd["owner"]).all()
    d = P.extract_dual_mesh(idx)
    base, lev = P.dual_bases(idx, d.tasks)
    assert (recs["base"] == base).all() and (recs["level"] == lev).all()
    ref.free(h)
