import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def orc():
    from oracle.cpu import Oracle
    return Oracle("orc")


@pytest.fixture(scope="session")
def ref():
    from oracle.cpu import Oracle, available
    if not available("ref"):
        pytest.skip("oracle/_ref not built (reference sources absent when building)")
    return Oracle("ref")


@pytest.fixture(scope="session")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_2006_06608_b200.capi import Context
    return Context(0)


def random_graph(rng, n, e, symmetrize=True, orc=None):
    """Reference helpers.hpp random_edges-style graph (duplicates and self
    loops allowed), canonicalised through the oracle's to_csr."""
    from oracle.cpu import Oracle
    o = orc or Oracle("orc")
    edges = rng.integers(0, n, size=(e, 2)).astype(np.uint32)
    rp, col = o.to_csr(n, edges, symmetrize)
    return rp, col, edges


def to_dev(*arrs):
    import torch
    out = []
    for a in arrs:
        t = torch.from_numpy(np.ascontiguousarray(a))
        if t.dtype == torch.uint64:
            t = t.view(torch.int64)
        elif t.dtype == torch.uint32:
            t = t.view(torch.int32)
        out.append(t.cuda())
    return out if len(out) > 1 else out[0]


class _Golden:
    """tests/golden/ref_golden.npz (reference-produced vectors)."""

    def __init__(self, path):
        self.z = np.load(path)
        self.keys = set(self.z.files)

    def __getitem__(self, k):
        return self.z[k]

    def ids(self, group):
        return sorted({int(k.split("/")[1]) for k in self.keys if k.startswith(group + "/")})


_GOLDEN = None


def golden_cases():
    global _GOLDEN
    if _GOLDEN is None:
        _GOLDEN = _Golden(os.path.join(ROOT, "tests", "golden", "ref_golden.npz"))
    return _GOLDEN
