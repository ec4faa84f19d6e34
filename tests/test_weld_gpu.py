"""GPU weld (amrx_weld, csrc/weld.cu) against the reference's weld
(proj/src/weld.cpp:31-64): the restatement (oracle/amrx_oracle.c orc_weld)
and, where it was built, the reference library itself.  Bit-exact vertex
arrays (position-sorted) and identical triangle indices."""
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
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2004_08475_b200 as P
    return P


def same(a, b):
    return a.shape == b.shape and (np.ascontiguousarray(a).view(np.uint64) ==
                                   np.ascontiguousarray(b).view(np.uint64)).all()


@pytest.mark.parametrize("name", sorted(CASES))
def test_weld_matches_restatement(P, name):
    fat = CASES[name]["fat"]
    m = P.weld(fat)
    v, t = oracles.restatement().weld(fat)
    assert same(m.vertices, v)
    assert (m.triangles == t).all()
    # expanding the indexed mesh gives the soup back (weld keeps triangle
    # order and exact positions)
    if len(fat):
        assert same(m.vertices[m.triangles.astype(np.int64)].reshape(-1, 9), fat)


def test_weld_matches_reference_library(P):
    R = oracles.reference()
    if R is None:
        pytest.skip("oracle/_ref not built")
    for name in ("octree_sphere", "slots_l4_s3", "blocks_jump2"):
        fat = CASES[name]["fat"]
        m = P.weld(fat)
        v, t = R.weld(fat)
        assert same(m.vertices, v) and (m.triangles == t).all()


def test_weld_device_input_and_larger_soup(P):
    """a ~1M-triangle soup of the brick generator, from a device tensor"""
    import torch
    from paper_2004_08475_b200 import synth
    ds = synth.bricks([24, 16, 16], seed=5, shuffle=True)
    idx = P.build_index(ds.cells, ds.scalars)
    fat = P.extract_isosurface(idx, P.IsoParams(iso=synth.C4_ISO)).fat
    idx.close()
    m = P.weld(torch.from_numpy(fat).cuda())  # the mesh stays on the device
    v, t = oracles.restatement().weld(fat)
    assert m.vertices.is_cuda and m.triangles.is_cuda
    assert same(m.vertices.cpu().numpy(), v)
    assert (m.triangles.cpu().numpy().view(np.uint32) == t).all()


def test_weld_empty(P):
    m = P.weld(np.zeros((0, 9)))
    assert m.vertices.shape == (0, 3) and m.triangles.shape == (0, 3)


def test_weld_signed_zero_is_one_vertex(P):
    """-0.0 == +0.0 in the reference's comparison: one vertex"""
    tri = np.array([[0.0, 1, 2, 3, 4, 5, 6, 7, 8], [-0.0, 1, 2, 9, 9, 9, 6, 7, 8]])
    m = P.weld(tri)
    v, t = oracles.restatement().weld(tri)
    assert same(m.vertices, v) and (m.triangles == t).all()


def test_weld_signed_zero_lowest_tag_keeps_its_bits(P):
    """the vertex carries the bits of the group's lowest-tag corner (-0.0 here)"""
    tri = np.array([[-0.0, 1, 2, 3, 4, 5, 6, 7, 8], [0.0, 1, 2, 9, 9, 9, 6, 7, 8],
                    [0.0, 1, -0.0, 3, 4, 5, 0, 0, 0]])
    m = P.weld(tri)
    v, t = oracles.restatement().weld(tri)
    assert same(m.vertices, v) and (m.triangles == t).all()
    assert np.signbit(m.vertices[m.triangles[0, 0], 0])  # (-0, 1, 2): tag 0 wins over tag 3


def test_weld_heavy_sharing(P):
    """200k triangles over 64 distinct positions (long groups, hash pressure),
    with signed zeros mixed in"""
    rng = np.random.default_rng(11)
    pts = rng.integers(-2, 3, size=(64, 3)).astype(np.float64)
    pick = rng.integers(0, 64, size=(200_000, 3))
    tri = pts[pick].reshape(-1, 9).copy()
    flip = (tri == 0) & (rng.random(tri.shape) < 0.5)
    tri[flip] = -0.0
    m = P.weld(tri)
    v, t = oracles.restatement().weld(tri)
    assert same(m.vertices, v) and (m.triangles == t).all()


def test_weld_sort_path_matches(P, tmp_path):
    """the sort-based GPU weld (AMRX_WELD=sort, read once per process) gives
    the same mesh as the hash weld"""
    import subprocess
    import sys
    from paper_2004_08475_b200 import synth
    ds = synth.bricks([16, 12, 12], seed=7, shuffle=True)
    idx = P.build_index(ds.cells, ds.scalars)
    fat = P.extract_isosurface(idx, P.IsoParams(iso=synth.C4_ISO)).fat
    idx.close()
    np.save(tmp_path / "fat.npy", fat)
    m = P.weld(fat)
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_2004_08475_b200 as P; "
            "m = P.weld(np.load(%r)); np.save(%r, m.vertices); np.save(%r, m.triangles)"
            % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
               str(tmp_path / "fat.npy"), str(tmp_path / "v.npy"), str(tmp_path / "t.npy")))
    subprocess.run([sys.executable, "-c", code], check=True, timeout=600,
                   env=dict(os.environ, AMRX_WELD="sort"))
    assert same(m.vertices, np.load(tmp_path / "v.npy"))
    assert (m.triangles == np.load(tmp_path / "t.npy")).all()


@pytest.mark.parametrize("name", ["slots_l4_s3", "octree_sphere", "acceptance_1"])
def test_extract_isosurface_mesh_equals_reference(P, ref, name):
    """extract + weld on the device (amrx_extract_iso_mesh, what the drop-in's
    extract_isosurface returns) == the reference's welded mesh, bit for bit"""
    import os
    here = os.path.dirname(os.path.abspath(__file__))
    z = np.load(os.path.join(here, "golden", "cases.npz"))
    cells, scal, iso = z[name + "/in_cells"], z[name + "/in_scalars"], float(z[name + "/iso"])
    idx = P.build_index(cells, scal)
    mesh, st, tw = P.extract_isosurface_mesh(idx, iso)
    h = ref.build(cells, scal)
    ri = ref.extract_iso(h, iso, 0)
    assert st.fat_triangle_count == ri["stats"]["fat_triangle_count"]
    assert mesh.vertices.shape == ri["verts"].shape
    assert (mesh.vertices.view(np.uint64) == ri["verts"].view(np.uint64)).all()
    assert (mesh.triangles == ri["tris"]).all()
    # a second call reuses the cached soup and mesh
    mesh2, _, _ = P.extract_isosurface_mesh(idx, iso)
    assert (mesh2.triangles == mesh.triangles).all()
    ref.free(h)
