"""CPU tests of the drop-in boundary: libamrx.so loads, exports every symbol
include/amrx.h declares, the Python mirror imports, and -- with no GPU --
every compute entry fails loudly instead of falling back to the CPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "amrx.h")
LIB = os.path.join(ROOT, "paper_2004_08475_b200", "libamrx.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*AMRX_API\s+(?:amrx_status|const char \*|uint64_t|void)\s*(amrx_\w+)\(", text,
                                 re.MULTILINE)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("amrx_index_create", "amrx_extract_dual", "amrx_extract_iso", "amrx_snap",
                 "amrx_find_exact", "amrx_try_build_duals", "amrx_index_adopt",
                 "amrx_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "libamrx.so not built"
    lib = C.CDLL(LIB)
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_library_exports_nothing_else():
    """-fvisibility=hidden: the C ABI is the whole dynamic surface"""
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True,
                         text=True).stdout
    amrx = sorted({ln.split()[-1] for ln in out.splitlines() if " T amrx_" in ln})
    assert amrx == declared_symbols()


def test_python_mirror_imports():
    import paper_2004_08475_b200 as P
    assert P.library() is not None
    assert P.library().amrx_version().decode().startswith("amrx")


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2004_08475_b200 as P
    with pytest.raises((P.CudaError, RuntimeError)):
        P.build_index(np.array([[0, 0, 0, 0]], np.int32), np.array([1.0]))


def test_argument_errors_precede_device_use():
    """build_index's input checks (locator.cpp:29-36) fire with reference
    wording even before a device is touched"""
    import paper_2004_08475_b200 as P
    with pytest.raises(P.LoadError, match="dataset is empty"):
        P.build_index(np.zeros((0, 4), np.int32), np.zeros(0))
    with pytest.raises(P.LoadError, match="cell count 1 does not match scalar count 2"):
        P.build_index(np.array([[0, 0, 0, 0]], np.int32), np.array([1.0, 2.0]))
