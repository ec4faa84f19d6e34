"""amrx_read_amr (read_amr, io.cpp:76-181): AMRCELL1 files through pinned
chunks to the GPU.  The index read from a file must equal build_index over
the same arrays; malformed files raise LoadError with the reference's
messages (test_io.cpp:135-236 pins the same wording through the drop-in)."""
import os
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2004_08475_b200 as P
    return P


def soup(n_side, seed):
    rng = np.random.default_rng(seed)
    g = np.stack(np.meshgrid(*[np.arange(n_side)] * 3, indexing="ij"), -1).reshape(-1, 3)
    cells = np.concatenate([g, np.zeros((len(g), 1), int)], 1).astype(np.int32)
    perm = rng.permutation(len(cells))
    return cells[perm], rng.normal(size=len(cells))


def same_index(a, b):
    assert (a.cells == b.cells).all()
    assert (a.scalars.view(np.uint64) == b.scalars.view(np.uint64)).all()
    assert list(a.levels) == list(b.levels) and a.bounds == b.bounds


def test_binary_round_trip_multi_chunk(P, tmp_path):
    cells, scal = soup(140, 5)  # 2.74M records: three 1M-record chunks, ragged tail
    path = tmp_path / "c.amr"
    P.write_amr(path, cells, scal)
    a = P.read_amr(path)
    b = P.build_index(cells, scal)
    same_index(a, b)
    r1 = P.extract_isosurface(a, P.IsoParams(iso=0.3))
    r2 = P.extract_isosurface(b, P.IsoParams(iso=0.3))
    assert (r1.fat.view(np.uint64) == r2.fat.view(np.uint64)).all()


def test_text_file(P, tmp_path):
    path = tmp_path / "cells.txt"
    path.write_text("# header comment\n\n0 0 0 0 1.5   # inline comment\n   \t\n1 0 0 0 -2\n")
    ix = P.read_amr(path)
    c, s = ix.cells, ix.scalars
    assert c.tolist() == [[0, 0, 0, 0], [1, 0, 0, 0]] and s.tolist() == [1.5, -2.0]


def load_error(P, path):
    with pytest.raises(P.LoadError) as e:
        P.read_amr(path)
    msg = str(e.value)
    assert str(path) in msg
    return msg


def test_binary_errors(P, tmp_path):
    cells = np.array([[0, 0, 0, 0], [1, 0, 0, 0], [0, 1, 0, 0]], np.int32)
    good_path = tmp_path / "good.amr"
    P.write_amr(good_path, cells, [1.0, 2.0, 3.0])
    good = good_path.read_bytes()
    path = tmp_path / "bad.amr"

    def case(data, needle):
        path.write_bytes(data)
        assert needle in load_error(P, path)

    def patched(off, fmt, v):
        b = bytearray(good)
        b[off:off + struct.calcsize(fmt)] = struct.pack(fmt, v)
        return bytes(b)

    case(good[:10], "shorter than the 24-byte header")
    case(b"X" + good[1:], "bad magic, not a cell data file")
    case(patched(8, "<I", 2), "unsupported version 2")
    case(patched(20, "<I", 7), "expected exactly 1 field, file declares 7")
    case(patched(12, "<Q", 0), "file declares zero cells")
    case(patched(12, "<Q", 4), "truncated: header declares 4 cells but only 3 fit in the file")
    case(good + b"xyz", "3 trailing bytes after the last record")
    case(patched(24 + 24 + 16, "<d", float("nan")), "record 1: scalar is not finite")
    case(patched(24 + 12, "<i", 31), "record 0: level 31 out of range")
    # non-finite wins over an earlier build_index error (the reader checks first)
    b = bytearray(patched(24 + 12, "<i", 31))
    b[24 + 48 + 16:24 + 48 + 24] = struct.pack("<d", float("inf"))
    case(bytes(b), "record 2: scalar is not finite")
    assert "cannot open" in load_error(P, tmp_path / "absent.amr")


def test_first_non_finite_across_chunks(P, tmp_path):
    cells, scal = soup(110, 9)  # 1.33M records: two chunks
    scal[1_200_000] = np.inf
    scal[1_100_000] = np.nan
    path = tmp_path / "big.amr"
    P.write_amr(path, cells, scal)
    assert "record 1100000: scalar is not finite" in load_error(P, path)


def test_text_errors(P, tmp_path):
    path = tmp_path / "cells.txt"
    for text, needle in [
        ("0 0 0 0 1\n1 0 0\n", "line 2: expected 'i j k level scalar'"),
        ("0 0 0 0 1 9\n", "line 1: trailing characters '9'"),
        ("# c\n3000000000 0 0 0 1\n", "line 2: anchor out of 32-bit range"),
        ("0 0 0 31 1\n", "line 1: level 31 out of range"),
        ("0 0 0 0 nan\n", "line 1: expected"),
        ("1 0 0 1 0.5\n", "not a multiple"),
        ("# only comments\n\n", "empty"),
    ]:
        path.write_text(text)
        assert needle in load_error(P, path)


def test_too_many_cells_refused_before_staging(P, tmp_path):
    # a sparse file whose size matches a 2^32-record header: refused by the
    # 32-bit CellId limit without reading or staging ~100 GB
    n = 1 << 32
    path = tmp_path / "huge.amr"
    with open(path, "wb") as f:
        f.write(b"AMRCELL1" + struct.pack("<IQI", 1, n, 1))
    os.truncate(path, 24 + 24 * n)
    assert "dataset too large for 32-bit cell ids" in load_error(P, path)
