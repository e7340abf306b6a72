import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA product path)")
    config.addinivalue_line("markers", "slow: long-running GPU parity case")


@pytest.fixture(scope="session")
def chk():
    """The C restatement of the reference (test-only checker)."""
    import oracle as O
    return O.restated()


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference library, when it was built (oracle/_ref)."""
    import oracle as O
    if not O.reference_available():
        pytest.skip("oracle/_ref/libnqref.so not built (needs /root/reference at build time)")
    return O.reference()


@pytest.fixture(scope="session")
def nq():
    import paper_2602_06694_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def ctx(nq):
    return nq.context(0)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


def bits_of(words: np.ndarray, cols: int) -> np.ndarray:
    """(rows, wpr) uint32 LSB-first -> (rows, cols) bool."""
    w = np.ascontiguousarray(words, dtype="<u4")
    b = np.unpackbits(w.view(np.uint8), axis=1, bitorder="little")
    return b[:, :cols].astype(bool)
