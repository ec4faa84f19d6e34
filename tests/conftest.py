import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ref():
    import oracles
    r = oracles.reference()
    if r is None:
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return r


@pytest.fixture(scope="session")
def orc():
    import oracles
    return oracles.restatement()


LOOKUPS = ["auto", "hash", "directory"]


class LookupProxy:
    """the package with build_index / read_amr / adopt_index defaulting to
    one lookup structure, so a whole parity module runs once per structure
    (dense records, hashed records, bucket directory) -- every choice must
    give bit-identical results"""

    def __init__(self, P, mode):
        self._P = P
        self.lookup_mode = None if mode == "auto" else mode

    def __getattr__(self, name):
        return getattr(self._P, name)

    def build_index(self, *a, **k):
        k.setdefault("lookup", self.lookup_mode)
        idx = self._P.build_index(*a, **k)
        if self.lookup_mode and idx.info.duplicate_keys == 0 and idx.info.key_bits <= 64:
            assert idx.info.lookup == self.lookup_mode, (idx.info.lookup, self.lookup_mode)
        return idx

    def read_amr(self, *a, **k):
        k.setdefault("lookup", self.lookup_mode)
        return self._P.read_amr(*a, **k)
