import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: larger CPU cases")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def rng():
    return np.random.default_rng(200606052)


def random_bsr(rng, n, b, density=0.3, m=None, diag=True, symmetric_pattern=False, dom=0.0):
    """Random BSR (ptr, col, val[nnz,b,b]) with sorted unique columns (test input only)."""
    m = n if m is None else m
    mask = rng.random((n, m)) < density
    if diag:
        for i in range(min(n, m)):
            mask[i, i] = True
    if symmetric_pattern and n == m:
        mask = mask | mask.T
    ptr = np.zeros(n + 1, dtype=np.int32)
    cols = []
    for i in range(n):
        c = np.nonzero(mask[i])[0]
        cols.append(c)
        ptr[i + 1] = ptr[i] + len(c)
    col = np.concatenate(cols).astype(np.int32) if cols else np.zeros(0, np.int32)
    val = rng.standard_normal((len(col), b, b))
    if dom:
        for i in range(n):
            for k in range(ptr[i], ptr[i + 1]):
                if col[k] == i:
                    val[k] += dom * np.eye(b)
    return ptr, col, val


def bsr_dense(ptr, col, val, m=None):
    n = len(ptr) - 1
    b = val.shape[-1]
    m = n if m is None else m
    D = np.zeros((n * b, m * b))
    for i in range(n):
        for k in range(ptr[i], ptr[i + 1]):
            D[i * b:(i + 1) * b, col[k] * b:(col[k] + 1) * b] += val[k]
    return D


def poisson1d(n):
    """1-D Poisson (2,-1) as b=1 BSR."""
    ptr = [0]
    col, val = [], []
    for i in range(n):
        for j in (i - 1, i, i + 1):
            if 0 <= j < n:
                col.append(j)
                val.append(2.0 if j == i else -1.0)
        ptr.append(len(col))
    return (np.array(ptr, np.int32), np.array(col, np.int32), np.array(val).reshape(-1, 1, 1))


def laplace3_blocks(n, b=3, noise=None):
    """7-point Laplacian (6,-1) tensor I_b on n^3 as BSR (zero row sums in the interior)."""
    import gen
    ptr, col, _ = gen.matrix(gen.POISSON3, n)
    val = np.zeros((len(col), b, b))
    for i in range(n ** 3):
        for k in range(ptr[i], ptr[i + 1]):
            val[k] = (6.0 if col[k] == i else -1.0) * np.eye(b)
    return ptr, col, val


@pytest.fixture
def envvars():
    """Set library tuning switches (read at plan / launch time) for one test."""
    saved = {}

    def set_(**kv):
        for k, v in kv.items():
            saved.setdefault(k, os.environ.get(k))
            os.environ[k] = str(v)
    yield set_
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
