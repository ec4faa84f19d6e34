"""GPU validate_dataset (amrx_validate, csrc/validate.cu) against the
reference library's validate_dataset (proj/src/locator.cpp:136-161): the
duplicate and overlap pair lists, in order, on valid and deliberately broken
datasets (duplicates and finer-inside-coarser overlaps mixed in)."""
import os

import numpy as np
import pytest

import oracles
from conftest import LOOKUPS, LookupProxy

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _cases():
    z = np.load(os.path.join(HERE, "golden", "cases.npz"))
    names = sorted({k.split("/")[0] for k in z.files})
    return {n: {k.split("/")[1]: z[k] for k in z.files if k.startswith(n + "/")} for n in names}


CASES = _cases()


@pytest.fixture(scope="module", params=LOOKUPS)
def env(request):
    """(package once per lookup structure, reference library)"""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    R = oracles.reference()
    if R is None:
        pytest.skip("oracle/_ref not built")
    import paper_2004_08475_b200 as P
    return LookupProxy(P, request.param), R


def broken(cells, scal, seed, n_dup=7, n_ovl=11):
    """duplicates of random cells + coarser cells enclosing random cells"""
    rng = np.random.default_rng(seed)
    extra_c, extra_s = [], []
    for i in rng.integers(0, len(cells), n_dup):
        extra_c.append(cells[i])
        extra_s.append(scal[i] + 1.0)
    lv_max = int(cells[:, 3].max())
    for i in rng.integers(0, len(cells), n_ovl):
        c = cells[i].copy()
        L = min(int(c[3]) + 1 + int(rng.integers(0, 2)), lv_max + 1)
        m = ~((1 << L) - 1)
        extra_c.append(np.array([c[0] & m, c[1] & m, c[2] & m, L], np.int32))
        extra_s.append(0.5)
    cc = np.concatenate([cells, np.array(extra_c, np.int32)])
    ss = np.concatenate([scal, np.array(extra_s)])
    p = rng.permutation(len(cc))
    return np.ascontiguousarray(cc[p]), np.ascontiguousarray(ss[p])


def check(P, R, cells, scal):
    idx = P.build_index(cells, scal)
    rep = P.validate_dataset(idx)
    h = R.build(cells, scal)
    dup, ovl = R.validate_pairs(h)
    assert rep.duplicates.shape == dup.shape and (rep.duplicates == dup).all()
    assert rep.overlaps.shape == ovl.shape and (rep.overlaps == ovl).all()
    R.free(h)
    return rep, idx


@pytest.mark.parametrize("name", sorted(CASES))
def test_valid_golden_cases(env, name):
    P, R = env
    c = CASES[name]
    rep, _ = check(P, R, c["in_cells"], c["in_scalars"])


@pytest.mark.parametrize("name,seed", [("slots_l4_s3", 1), ("octree_sphere", 2),
                                       ("blocks_jump2", 3), ("acceptance_34", 4)])
def test_broken_datasets(env, name, seed):
    P, R = env
    c = CASES[name]
    cells, scal = broken(c["in_cells"], c["in_scalars"], seed)
    rep, idx = check(P, R, cells, scal)
    assert len(rep.duplicates) >= 1 and len(rep.overlaps) >= 1
    assert not rep.ok()
    text = rep.describe(idx)
    assert text.startswith(f"{len(rep.duplicates)} duplicate pair(s), ")
