"""The drop-in proof: the reference's OWN unit tests (65 cases) and
acceptance criteria (9), compiled unmodified and linked against the GPU shim
(paper_2004_08475_b200/shim/amriso_gpu.cpp -> libamrx.so) in place of the
reference's build_index / extract_isosurface / extract_dual_mesh.

Expected outcome equals the reference's own run (oracle/_ref/amriso_tests,
amriso_acceptance): all unit cases pass; acceptance passes 8 of 9, the one
failure being the PLY golden that the reference tree does not ship
(acceptance.cpp:417).  The binaries are built where
/root/reference exists (`make -C oracle gpu-tests`) and travel prebuilt."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")


def run(name, timeout=600):
    path = os.path.join(REF, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not built (needs /root/reference at build time)")
    p = subprocess.run([path], capture_output=True, text=True, timeout=timeout, cwd=REF)
    return p.returncode, p.stdout + p.stderr


def summary(text):
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", text)
    assert m, text[-2000:]
    return tuple(int(x) for x in m.groups())


@pytest.fixture(scope="module")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_reference_unit_tests_on_gpu(gpu):
    rc, out = run("amriso_tests_gpu")
    total, passed, failed = summary(out)
    assert (total, failed) == (65, 0), out[-3000:]


def test_reference_acceptance_on_gpu(gpu):
    rc, out = run("amriso_acceptance_gpu")
    total, passed, failed = summary(out)
    lines = [ln for ln in out.splitlines() if ln.startswith("[")]
    fails = [ln for ln in lines if ln.startswith("[FAIL]")]
    # identical to the reference's own result: only the unshipped PLY golden
    assert total == 9 and failed == 1, out[-3000:]
    assert len(fails) == 1 and "ply DIFFERS" in fails[0] and "obj stable" in fails[0]
    for must in ("100 datasets, 68934 dual cells", "102 datasets, 74877 dual cells, 0 duplicates",
                 "102 datasets, 116719 triangles, 0 disagreements",
                 "16^3: 480 vertices equal, 32^3: 1896 vertices equal",
                 "0 boundary, 0 overshared"):
        assert any(must in ln for ln in lines), (must, lines)
