"""Single-process multi-GPU C ABI (amrx_comm_*, csrc/comm.cu): a comm over
every visible device (one on the test box), the index built on the first
device and broadcast with NCCL, each device extracting its share.  The
concatenated output must equal the single-GPU extraction bit for bit, for
host and device outputs, and the drop-in shim's multi-GPU path (AMRISO_GPUS)
runs the reference's own tests."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _cases():
    z = np.load(os.path.join(HERE, "golden", "cases.npz"))
    names = sorted({k.split("/")[0] for k in z.files})
    return {n: {k.split("/")[1]: z[k] for k in z.files if k.startswith(n + "/")} for n in names}


CASES = _cases()


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2004_08475_b200 as P
    return P


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


@pytest.mark.parametrize("name", ["slots_l4_s3", "octree_sphere", "acceptance_1"])
def test_comm_matches_single_gpu(P, name):
    c = CASES[name]
    comm = P.Comm()
    assert comm.size() == P.device_count() >= 1
    m = comm.build_index(c["in_cells"], c["in_scalars"])
    r = m.extract_isosurface(P.IsoParams(iso=float(c["iso"])))
    assert (bits(r.fat) == bits(c["fat"])).all()
    s = r.stats
    assert [s.duals_accepted, s.duals_missing_corner, s.duals_finer_corner,
            s.duals_lower_key_corner] == [int(x) for x in c["counters"]]
    d = m.extract_dual_mesh()
    assert (d.corners == c["dual_corners"]).all() and (d.tasks == c["dual_tasks"]).all()
    m.close()
    comm.close()


def test_comm_device_output_and_capacity(P):
    import torch
    c = CASES["slots_l4_s3"]
    comm = P.Comm([0])
    m = comm.build_index(c["in_cells"], c["in_scalars"], lookup="hash")
    out = torch.empty((len(c["fat"]), 9), dtype=torch.float64, device="cuda")
    r = m.extract_isosurface(P.IsoParams(iso=float(c["iso"])), out=out)
    assert (bits(r.fat.cpu().numpy()) == bits(c["fat"])).all()
    small = np.empty((3, 9), np.float64)
    with pytest.raises(P.CapacityError) as e:
        m.extract_isosurface(P.IsoParams(iso=float(c["iso"])), out=small)
    assert e.value.count == len(c["fat"])
    with pytest.raises(ValueError):
        P.Comm([0, 0])  # a device listed twice


def test_comm_init_rejects_missing_device(P):
    with pytest.raises(ValueError):
        P.Comm([P.device_count() + 3])
