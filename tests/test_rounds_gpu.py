"""Extraction rounds (csrc/extract.cu run_extract): the staging buffers
only decide how many rounds a call takes, never the result.  With the
per-round staging capped (amrx_debug_round_limit) small datasets run in many
rounds; every output -- duals, task ids, the FP64 soup, counters -- must equal
the single-round result and the golden vectors, for device, pinned-host and
pageable-host outputs and for every lookup structure."""
import os

import numpy as np
import pytest

from conftest import LOOKUPS, LookupProxy

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _cases():
    z = np.load(os.path.join(HERE, "golden", "cases.npz"))
    names = sorted({k.split("/")[0] for k in z.files})
    return {n: {k.split("/")[1]: z[k] for k in z.files if k.startswith(n + "/")} for n in names}


CASES = _cases()


@pytest.fixture(scope="module", params=LOOKUPS)
def P(request):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2004_08475_b200 as P
    yield LookupProxy(P, request.param)
    P.debug_round_limit(0)


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("limit", [1, 37, 1000])
@pytest.mark.parametrize("name", ["slots_l4_s3", "octree_sphere", "blocks_jump2",
                                  "acceptance_1"])
def test_many_rounds_equal_golden(P, name, limit):
    c = CASES[name]
    P.debug_round_limit(limit)
    try:
        idx = P.build_index(c["in_cells"], c["in_scalars"])
        d = P.extract_dual_mesh(idx)
        assert (d.corners == c["dual_corners"]).all()
        assert (d.tasks == c["dual_tasks"]).all()
        r = P.extract_isosurface(idx, P.IsoParams(iso=float(c["iso"])))
        assert r.fat.shape == c["fat"].shape
        assert (bits(r.fat) == bits(c["fat"])).all()
        s = r.stats
        assert [s.duals_accepted, s.duals_missing_corner, s.duals_finer_corner,
                s.duals_lower_key_corner] == [int(x) for x in c["counters"]]
    finally:
        P.debug_round_limit(0)


@pytest.mark.parametrize("limit", [1, 500])
def test_rounds_device_and_pinned_outputs(P, limit):
    import torch
    c = CASES["slots_l4_s3"]
    P.debug_round_limit(limit)
    try:
        idx = P.build_index(c["in_cells"], c["in_scalars"])
        nt, nd = len(c["fat"]), len(c["dual_corners"])
        for pin in (False, True):
            kw = dict(pin_memory=True) if pin else dict(device="cuda")
            fat = torch.empty((nt, 9), dtype=torch.float64, **kw)
            r = P.extract_isosurface(idx, P.IsoParams(iso=float(c["iso"])), out=fat)
            assert (bits(r.fat.cpu().numpy()) == bits(c["fat"])).all()
            cor = torch.empty((nd, 8), dtype=torch.int32, **kw)
            tsk = torch.empty(nd, dtype=torch.int64, **kw)
            d = P.extract_dual_mesh(idx, out=(cor, tsk))
            assert (d.corners.cpu().numpy().view(np.uint32) == c["dual_corners"]).all()
            assert (d.tasks.cpu().numpy().view(np.uint64) == c["dual_tasks"]).all()
        # a buffer one triangle short: capacity error with the full count,
        # and every triangle that fits is still written in order
        short = torch.empty((nt - 1, 9), dtype=torch.float64, device="cuda")
        with pytest.raises(P.CapacityError) as e:
            P.extract_isosurface(idx, P.IsoParams(iso=float(c["iso"])), out=short)
        assert e.value.count == nt
        assert (bits(short.cpu().numpy()) == bits(c["fat"][: nt - 1])).all()
    finally:
        P.debug_round_limit(0)


def test_rounds_launch_more_kernels(P):
    c = CASES["slots_l4_s3"]
    idx = P.build_index(c["in_cells"], c["in_scalars"])
    one = P.extract_isosurface(idx, P.IsoParams(iso=float(c["iso"]))).stats.kernel_launches
    P.debug_round_limit(64)
    try:
        idx2 = P.build_index(c["in_cells"], c["in_scalars"])
        many = P.extract_isosurface(idx2, P.IsoParams(iso=float(c["iso"]))).stats
    finally:
        P.debug_round_limit(0)
    assert many.kernel_launches > one
    assert many.fat_triangle_count == len(c["fat"])
