"""Seeded synthetic inputs for the five configurations of BASELINE.json.

The reference and the paper both measure on synthetic keys; these recipes
 stand in for them.  Every generator is a pure function of
its config id, so the golden fixtures, the parity tests and ``bench.py`` all
see the same bytes.

* C1: 2,000 leaves x n=16, plain search   (``default_rng(1)``)
* C2: N=100,000 keys, n=24, b=500, rotate  (``default_rng(2)``), 1e6 queries (``default_rng(1002)``)
* C3: 100,000 leaves x n=32, plain         (``default_rng(3)``)
* C4: N=10,000,000 keys, n=40, b=2000      (``default_rng(4)``), 1e8 queries (``default_rng(1004)``)
* C5: 20,000 leaves x n=56, plain          (``default_rng(5)``); the 128-bit
  fingerprints are used directly as the (hi, lo) master hash code.
"""

import numpy as np

LEAF_CONFIGS = {
    1: dict(leaves=2000, n=16),
    3: dict(leaves=100_000, n=32),
    5: dict(leaves=20_000, n=56),
}

BUILD_CONFIGS = {
    2: dict(N=100_000, n=24, b=500, queries=1_000_000, qseed=1002),
    4: dict(N=10_000_000, n=40, b=2000, queries=100_000_000, qseed=1004),
}


def raw_keys(cfg: int, count: int) -> np.ndarray:
    """Uniform random 64-bit integer keys, ``default_rng(cfg)``."""
    rng = np.random.default_rng(cfg)
    return rng.integers(0, 2**64, count, dtype=np.uint64)


def keys_as_bytes(k: np.ndarray):
    """8-byte little-endian byte strings (``struct.pack('<Q', k)``)."""
    blob = np.ascontiguousarray(k, dtype="<u8").tobytes()
    return [blob[i : i + 8] for i in range(0, len(blob), 8)]


def keys_as_blob(k: np.ndarray):
    """Same keys as a packed byte blob plus CSR offsets (the C-ABI layout)."""
    blob = np.frombuffer(np.ascontiguousarray(k, dtype="<u8").tobytes(), dtype=np.uint8)
    offs = np.arange(0, 8 * (len(k) + 1), 8, dtype=np.int64)
    return blob, offs


def leaf_inputs(cfg: int, leaves: int = None):
    """(hi, lo) uint64 arrays of shape [leaves, n] for a leaf-only config.

    C1/C3: keys -> 8-byte LE strings -> blake2b-128 master hash (salt 0).
    C5: ``fp = rng.integers(0, 2**64, (L, 56, 2))`` used directly as (hi, lo).
    ``leaves`` takes a prefix sample (same leaves as the full config).
    """
    spec = LEAF_CONFIGS[cfg]
    L, n = spec["leaves"], spec["n"]
    if cfg == 5:
        rng = np.random.default_rng(5)
        fp = rng.integers(0, 2**64, (L, n, 2), dtype=np.uint64)
        hi = np.ascontiguousarray(fp[..., 0])
        lo = np.ascontiguousarray(fp[..., 1])
    else:
        k = raw_keys(cfg, L * n)
        hi, lo = blake2b_host(keys_as_bytes(k), 0)
        hi = hi.reshape(L, n)
        lo = lo.reshape(L, n)
    if leaves is not None:
        hi, lo = hi[:leaves], lo[:leaves]
    return np.ascontiguousarray(hi), np.ascontiguousarray(lo)


def blake2b_host(keys, salt: int = 0):
    """hashlib blake2b-128 fingerprints, used ONLY to synthesize inputs.

    The product path fingerprints on the GPU (``keys.master_hash_many``);
    this helper exists so input recipes do not need a GPU.
    """
    import hashlib
    import struct

    salt_b = struct.pack("<QQ", salt & 0xFFFFFFFFFFFFFFFF, 0)
    out = np.empty((len(keys), 2), dtype=np.uint64)
    for i, key in enumerate(keys):
        out[i] = struct.unpack("<QQ", hashlib.blake2b(key, digest_size=16, salt=salt_b).digest())
    return np.ascontiguousarray(out[:, 0]), np.ascontiguousarray(out[:, 1])


def build_keys(cfg: int) -> np.ndarray:
    """The N unique raw 64-bit keys of a build config (asserted unique)."""
    spec = BUILD_CONFIGS[cfg]
    k = raw_keys(cfg, spec["N"])
    if len(np.unique(k)) != len(k):
        raise AssertionError("synthetic keys are not unique")
    return k


def query_indices(cfg: int, count: int = None) -> np.ndarray:
    spec = BUILD_CONFIGS[cfg]
    count = spec["queries"] if count is None else count
    return np.random.default_rng(spec["qseed"]).integers(0, spec["N"], count)
