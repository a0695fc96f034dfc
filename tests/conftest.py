import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA kernels)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def K():
    from paper_2308_09561_b200._kernels import kernels

    return kernels


def hashed_leaf(n, gen_seed):
    from paper_2308_09561_b200.keys import HashedKey, synthetic_hashed

    hi, lo = synthetic_hashed(n, gen_seed)
    return [HashedKey(int(a), int(b)) for a, b in zip(hi, lo)]


def full_leaf_golden(cfg):
    """(seeds i64[L], fbits u64[L], passes u64[L], meta) of every leaf of a
    leaf-only config, made by the reference's compiled search_plain + orient
    (tests/golden/make_leaf_full.py); the file's sha256 is checked."""
    import hashlib

    meta = golden(f"c{cfg}_full.json")
    with open(os.path.join(GOLDEN, f"c{cfg}_full.bin"), "rb") as f:
        raw = f.read()
    assert hashlib.sha256(raw).hexdigest() == meta["file_sha256"]
    L = meta["leaves"]
    a = np.frombuffer(raw, dtype="<u8")
    assert a.size == 3 * L
    return a[:L].view("<i8"), a[L : 2 * L], a[2 * L :], meta
