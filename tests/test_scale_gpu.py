"""Parity at the BASELINE.json sizes (GPU).

* C2 (~9.7M cells, block-structured, level jumps up to 4, holes, white
  noise, iso 0.1): FULL bit-exact comparison of the dual mesh, the reject
  counters and the FP64 soup against the reference library itself.
* C3 (105M-cell 6-level noise octree): FULL bit-exact comparison with the
  reference library too (slow: the reference's serial sort and weld).
* C3, C4 (626M-cell soup) and C5 (250M, dual mesh only): (a) the ingest
  loses and invents nothing -- an order-independent hash of the input
  (cell, scalar) pairs equals that of the sorted arrays, whose keys
  strictly increase; (b) sampled cell ranges covering >= 1% of the cells,
  including every 8-way partition boundary, are compared bit-for-bit with
  the C restatement evaluated over the SAME full index (candidates near a
  range edge see the whole index, exactly like the reference); (c)
  size-independent properties hold on the full output: candidate accounting
  (accepted+missing+finer+lower-key == 8N, pipeline.cpp:106-107), every
  dual emitted exactly once (distinct canonical corner multisets,
  acceptance.cpp:260-284), candidate order, and the partitioned extraction
  reassembling the full one."""
import numpy as np
import pytest

import oracles

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2004_08475_b200 as P
    return P


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def test_c2_full_bit_exact_vs_reference(P, ref):
    from paper_2004_08475_b200 import synth
    cells, scal = synth.slots(2026, 23, 4, 0.15)
    assert 9_000_000 < len(cells) < 10_500_000
    idx = P.build_index(cells, scal)
    h = ref.build(cells, scal)
    ds = ref.dataset(h)
    assert (idx.cells == ds.cells).all() and (bits(idx.scalars) == bits(ds.scalars)).all()
    assert idx.levels == ds.levels == [0, 1, 2, 3, 4]
    d = P.extract_dual_mesh(idx)
    rd = ref.extract_dual(h, 0)
    assert d.corners.shape == rd["corners"].shape and (d.corners == rd["corners"]).all()
    assert (d.owner == rd["owner"]).all()
    r = P.extract_isosurface(idx, P.IsoParams(iso=0.1))
    ri = ref.extract_iso(h, 0.1, 0)
    st = ri["stats"]
    assert [r.stats.duals_accepted, r.stats.duals_missing_corner, r.stats.duals_finer_corner,
            r.stats.duals_lower_key_corner] == [st["duals_accepted"], st["duals_missing_corner"],
                                                st["duals_finer_corner"],
                                                st["duals_lower_key_corner"]]
    assert r.fat.shape == ri["fat"].shape and (bits(r.fat) == bits(ri["fat"])).all()
    ref.free(h)


def test_synth_generators_match_reference(ref):
    """our host generators reproduce the reference's generators record for
    record (after build_index), so bench inputs are the reference's"""
    from paper_2004_08475_b200 import synth
    for args in [(7, 6, 4, 0.15), (3, 4, 2, 0.15)]:
        c, s = synth.slots(*args)
        h = ref.gen_slots(*args)
        ds = ref.dataset(h)
        o = oracles.restatement()
        ho = o.build(c, s)
        mine = o.dataset(ho)
        assert (mine.cells == ds.cells).all() and (bits(mine.scalars) == bits(ds.scalars)).all()
        o.free(ho)
        ref.free(h)
    c, s = synth.octree_sphere(6, (25.0, 27.5, 30.0), 20.0, 3.2)
    h = ref.gen_octree(6, "sphere", [25, 27.5, 30, 20.0], 3.2)
    ds = ref.dataset(h)
    o = oracles.restatement()
    ho = o.build(c, s)
    mine = o.dataset(ho)
    assert len(mine) == 126_771
    assert (mine.cells == ds.cells).all() and (bits(mine.scalars) == bits(ds.scalars)).all()


def pair_hash(cells, scal):
    """order-independent hash of (cell, scalar) pairs on the GPU: the
    wrapping sum of a mixed 64-bit word per pair"""
    import torch
    c = cells.to(torch.int64)
    s = scal.contiguous().view(torch.int64)
    h = torch.zeros(len(c), dtype=torch.int64, device=c.device)
    for col, mult in ((c[:, 0], 0x1F3D5B79), (c[:, 1], 0x2545F491), (c[:, 2], 0x3C6EF372),
                      (c[:, 3], 0x4F1BBCDD), (s, 0x5851F42D)):
        x = (h ^ col) * mult + 0x632BE59B
        h = x ^ (x >> 29)
    return int(h.sum().item())


def _big(P, name, keep_input=False):
    """the configuration's index, the input's pair hash (and the input)"""
    import gc
    import torch
    from paper_2004_08475_b200 import synth
    # the previous big test's tensors sit in torch's cache and its index may
    # not be collected yet: give the memory back before the next 100+ GB
    gc.collect()
    torch.cuda.empty_cache()
    P.release_cached_memory()
    cfg = synth.CONFIGS[name]
    if cfg["kind"] == "octree_noise":
        cells, scal = synth.octree_noise(*cfg["args"])
    else:
        b3 = cfg["bricks"]
        ds = synth.bricks(b3, seed=cfg["seed"], shuffle=cfg["shuffle"],
                          knobs=cfg.get("knobs", synth.C4_KNOBS), holes=synth.body_holes(b3))
        cells, scal = ds.cells, ds.scalars
    h_in = pair_hash(cells, scal)
    idx = P.build_index(cells, scal)
    inp = (cells.cpu().numpy(), scal.cpu().numpy()) if keep_input else None
    del cells, scal
    torch.cuda.synchronize()
    return idx, h_in, inp


def _check_ingest(idx, h_in):
    """nothing lost or invented by the sort, keys strictly increasing"""
    import torch
    c = torch.from_numpy(idx.cells).cuda()
    s = torch.from_numpy(idx.scalars).cuda()
    assert pair_hash(c, s) == h_in
    a, b = c[:-1].to(torch.int64), c[1:].to(torch.int64)
    gt = b[:, 3] > a[:, 3]
    for k in (2, 1, 0):
        gt = (b[:, k] > a[:, k]) | ((b[:, k] == a[:, k]) & gt)
    assert bool(gt.all().item())
    del c, s, a, b, gt
    torch.cuda.empty_cache()


def _oracle_over(idx):
    """the restatement over the GPU index's sorted arrays (presorted path)"""
    o = oracles.restatement()
    h = o.build(idx.cells, idx.scalars)
    return o, h


def _exactly_once(P, corners):
    """distinct canonical corner multisets, on the GPU, via two independent
    symmetric 64-bit hashes (a duplicate dual collides in both)"""
    import torch
    c = torch.as_tensor(corners).cuda() if not hasattr(corners, "cuda") else corners
    n = c.shape[0]
    hs = []
    for mult, add in ((0x9E3779B97F4A7C15, 0x632BE59BD9B4E019), (0xC2B2AE3D27D4EB4F, 0x165667B19E3779F9)):
        h = torch.zeros(n, dtype=torch.int64, device=c.device)
        for k in range(8):  # one widened column at a time (memory)
            x = (c[:, k].to(torch.int64) & 0xFFFFFFFF) * \
                (mult - (1 << 64) if mult >= 1 << 63 else mult) + add
            x = x ^ (x >> 29)
            x = x * 0x5851F42D4C957F2D
            x = x ^ (x >> 32)
            h = h + x
        hs.append(h)
    order = torch.argsort(hs[0])
    a, b = hs[0][order], hs[1][order]
    same = (a[1:] == a[:-1]) & (b[1:] == b[:-1])
    return int(same.sum().item())


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_full_scale_properties_and_sampled_parity(P, name):
    import torch
    idx, h_in, _ = _big(P, name)
    n = len(idx)
    assert n > {"c3": 99_000_000, "c4": 600_000_000, "c5": 240_000_000}[name]
    _check_ingest(idx, h_in)
    from paper_2004_08475_b200 import synth
    iso = synth.C4_ISO if synth.CONFIGS[name]["iso"] is None else synth.CONFIGS[name]["iso"]
    if name == "c3":
        assert idx.levels == [0, 1, 2, 3, 4, 5]
    # --- dual mesh on the device
    cap = int(n * (1.9 if name == "c3" else 1.2))  # octrees own ~1.7 duals per cell
    corners = torch.empty((cap, 8), dtype=torch.int32, device="cuda")
    tasks = torch.empty(cap, dtype=torch.int64, device="cuda")
    d = P.extract_dual_mesh(idx, out=(corners, tasks))
    s = d.stats
    nd = len(d.corners)
    assert s.duals_accepted + s.duals_missing_corner + s.duals_finer_corner + \
        s.duals_lower_key_corner == 8 * n
    assert nd == s.duals_accepted
    # candidate order: task ids strictly increasing (owner major, delta minor)
    t = d.tasks
    assert bool((t[1:] > t[:-1]).all().item())
    assert _exactly_once(P, d.corners) == 0
    del corners, tasks, d, t
    torch.cuda.empty_cache()
    # --- sampled bit-exact parity against the restatement over the same
    # index: >= 1% of the cells, every 8-way partition boundary inside a range
    o, h = _oracle_over(idx)
    rng = np.random.default_rng(2026)
    width = max(3000, n // 400)
    starts = [max(0, n * r // 8 - width // 2) for r in range(1, 8)]
    starts += sorted(rng.integers(0, n - width, 3).tolist()) + [0, n - width]
    assert len(starts) * width >= n // 100
    for b in starts:
        e = b + width
        gd = P.extract_dual_mesh(idx, cell_range=(b, e))
        od = o.extract_dual_range(h, b, e)
        assert (gd.corners == od["corners"]).all(), (name, b)
        assert (gd.owner == od["owner"]).all()
        if name != "c5":  # C5 is the dual-mesh-only configuration
            gi = P.extract_isosurface(idx, P.IsoParams(iso=iso), cell_range=(b, e))
            oi = o.extract_iso(h, iso, b, e)
            assert gi.fat.shape == oi["fat"].shape, (b, gi.fat.shape, oi["fat"].shape)
            assert (bits(gi.fat) == bits(oi["fat"])).all(), (name, b)
            assert [gi.stats.duals_accepted, gi.stats.duals_missing_corner,
                    gi.stats.duals_finer_corner, gi.stats.duals_lower_key_corner] == \
                [int(x) for x in oi["counters"]]
    o.free(h)


def test_c4_partitioned_equals_full(P):
    """4-way range partition, concatenated in rank order == the full soup
    (the multi-GPU contract), at full scale on one device"""
    import torch
    from paper_2004_08475_b200 import synth
    idx, _, _ = _big(P, "c4")
    n = len(idx)
    full = P.extract_isosurface(idx, P.IsoParams(iso=synth.C4_ISO))
    total = len(full.fat)
    digest = torch.from_numpy(bits(full.fat)).cuda()
    acc = 0
    for r in range(4):
        lo, hi = n * r // 4, n * (r + 1) // 4
        part = P.extract_isosurface(idx, P.IsoParams(iso=synth.C4_ISO), cell_range=(lo, hi))
        k = len(part.fat)
        assert (torch.from_numpy(bits(part.fat)).cuda() == digest[acc: acc + k]).all()
        acc += k
    assert acc == total
    # pinned host output takes the chunked, download-overlapped path
    host = torch.empty((total + 16, 9), dtype=torch.float64, pin_memory=True)
    h = P.extract_isosurface(idx, P.IsoParams(iso=synth.C4_ISO), out=host)
    assert len(h.fat) == total
    assert (torch.from_numpy(bits(h.fat.numpy())).cuda() == digest).all()
    # and a too-small pinned buffer reports the needed count
    small = torch.empty((total // 2, 9), dtype=torch.float64, pin_memory=True)
    with pytest.raises(P.CapacityError) as e:
        P.extract_isosurface(idx, P.IsoParams(iso=synth.C4_ISO), out=small)
    assert e.value.count == total


@pytest.mark.slow
def test_c3_full_bit_exact_vs_reference(P, ref):
    """C3 (104.8M cells, 6 levels) end to end against the reference library:
    the same shuffled input through both build_index, then every dual, the
    reject counters and the FP64 soup bit for bit ("full on
    <= 100M")"""
    from paper_2004_08475_b200 import synth
    idx, h_in, (cells, scal) = _big(P, "c3", keep_input=True)
    _check_ingest(idx, h_in)
    h = ref.build(cells, scal)
    del cells, scal
    ds = ref.dataset(h)
    assert (idx.cells == ds.cells).all() and (bits(idx.scalars) == bits(ds.scalars)).all()
    del ds
    d = P.extract_dual_mesh(idx)
    rd = ref.extract_dual(h, 0)
    assert d.corners.shape == rd["corners"].shape and (d.corners == rd["corners"]).all()
    assert (d.owner == rd["owner"]).all()
    del d, rd
    iso = synth.CONFIGS["c3"]["iso"]
    r = P.extract_isosurface(idx, P.IsoParams(iso=iso))
    ri = ref.extract_iso(h, iso, 0)
    st = ri["stats"]
    assert [r.stats.duals_accepted, r.stats.duals_missing_corner, r.stats.duals_finer_corner,
            r.stats.duals_lower_key_corner] == [st["duals_accepted"], st["duals_missing_corner"],
                                                st["duals_finer_corner"],
                                                st["duals_lower_key_corner"]]
    assert r.fat.shape == ri["fat"].shape and (bits(r.fat) == bits(ri["fat"])).all()
    ref.free(h)
