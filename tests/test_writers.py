"""Output writers (write_obj / write_ply / write_dual_mesh, io.cpp:212-305):
host code in libamrx.so, so these run on CPU.  Bytes must equal the
reference's own writers (oracle/_ref, where built) and the shipped golden
OBJ (tests/golden/sphere16.obj, acceptance.cpp:411-421)."""
import os

import numpy as np
import pytest

import oracles

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "sphere16.obj")


@pytest.fixture(scope="module")
def P():
    import paper_2004_08475_b200 as P
    return P


def ref_or_skip():
    R = oracles.reference()
    if R is None:
        pytest.skip("reference library not built (oracle/_ref)")
    return R


class Mesh:
    def __init__(self, v, t):
        self.vertices, self.triangles = v, t


def parse_obj(path):
    v, t = [], []
    for line in open(path):
        if line.startswith("v "):
            v.append([float(x) for x in line.split()[1:]])
        elif line.startswith("f "):
            t.append([int(x) - 1 for x in line.split()[1:]])
    return Mesh(np.array(v, np.float64), np.array(t, np.uint32))


def random_mesh(nv, nt, seed):
    rng = np.random.default_rng(seed)
    v = rng.normal(size=(nv, 3)) * 10.0 ** rng.integers(-8, 9, size=(nv, 1))
    v[::7] = np.round(v[::7])       # integral values print without a fraction
    v[1::11] = -0.0
    v[2::13] = 1e300
    v[3::17] = 5e-324               # denormal
    t = rng.integers(0, nv, size=(nt, 3)).astype(np.uint32)
    return Mesh(v, t)


def test_obj_golden_bytes(P, tmp_path):
    m = parse_obj(GOLDEN)
    out = tmp_path / "s.obj"
    P.write_obj(out, m, threads=3)
    assert out.read_bytes() == open(GOLDEN, "rb").read()
    assert not (tmp_path / "s.obj.tmp").exists()


@pytest.mark.parametrize("nv,nt", [(0, 0), (5, 3), (200_003, 150_001)])
def test_mesh_writers_match_reference(P, tmp_path, nv, nt):
    R = ref_or_skip()
    m = random_mesh(nv, nt, nv + nt)
    for ply in (0, 1):
        mine, ref = tmp_path / f"a{ply}", tmp_path / f"b{ply}"
        (P.write_ply if ply else P.write_obj)(mine, m, threads=8)
        assert R.lib.ref_write_mesh(os.fsencode(str(ref)), ply, oracles._ptr(m.vertices), nv,
                                    oracles._ptr(m.triangles), nt) == 0
        assert mine.read_bytes() == ref.read_bytes()


def test_dual_mesh_writer_matches_reference(P, tmp_path):
    R = ref_or_skip()
    rng = np.random.default_rng(4)
    nc = 5000
    lev = rng.integers(0, 4, nc)
    cells = np.stack([rng.integers(-1000, 1000, nc) << lev, rng.integers(-1000, 1000, nc) << lev,
                      rng.integers(0, 1000, nc) << lev, lev], 1).astype(np.int32)
    scal = rng.normal(size=nc)
    corners = rng.integers(0, nc, size=(70_001, 8)).astype(np.uint32)

    class Index:
        pass
    ix = Index()
    ix.cells, ix.scalars = cells, scal
    mine, ref = tmp_path / "a.txt", tmp_path / "b.txt"
    P.write_dual_mesh(mine, corners, ix, threads=5)
    assert R.lib.ref_write_dual_mesh(os.fsencode(str(ref)), oracles._ptr(corners), len(corners),
                                     oracles._ptr(cells), oracles._ptr(scal), nc) == 0
    assert mine.read_bytes() == ref.read_bytes()


def test_writer_errors(P, tmp_path):
    m = Mesh(np.zeros((2, 3)), np.array([[0, 1, 2]], np.uint32))
    with pytest.raises(ValueError, match="out of range"):
        P.write_obj(tmp_path / "x.obj", m)
    m = Mesh(np.zeros((3, 3)), np.array([[0, 1, 2]], np.uint32))
    with pytest.raises(OSError, match="cannot open .*x.obj.tmp for writing"):
        P.write_obj(tmp_path / "missing_dir" / "x.obj", m)
    target = tmp_path / "keep.obj"
    target.write_text("old")
    P.write_obj(target, m)
    assert target.read_text().startswith("# amriso mesh: 3 vertices, 1 triangles\n")
