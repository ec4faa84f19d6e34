"""bench.py's steady-state e2e (consecutive steps, each step's download
overlapping the next upload) moves the real soup: the last step's downloaded
triangles equal the device path's, bit for bit (C1, one B200)."""
import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_pipelined_e2e_downloads_the_soup():
    import torch
    import paper_2004_08475_b200 as P
    sys.path.insert(0, ROOT)
    import bench
    dev = torch.device("cuda", 0)
    cells, scal, _ = bench.make_workload("c1", dev)
    iso = bench.iso_of("c1")
    ix = P.build_index(cells, scal)
    ref = np.asarray(P.extract_isosurface(ix, P.IsoParams(iso=iso)).fat)
    ix.close()
    hcells = torch.empty(cells.shape, dtype=torch.int32, pin_memory=True)
    hscal = torch.empty(scal.shape, dtype=torch.float64, pin_memory=True)
    hcells.copy_(cells)
    hscal.copy_(scal)
    args = SimpleNamespace(steps=3, lookup=None)
    res = bench.e2e_pipelined(P, hcells, hscal, iso, len(ref) + 1024, len(cells), 0, None, args,
                              keep=True)
    assert res["triangles"] == len(ref) and res["steps"] >= 2 and res["ms_per_step"] > 0
    got = res["_soup"].numpy()
    assert got.shape == ref.shape
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
