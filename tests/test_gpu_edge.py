"""Edge cases of the whole build on the GPU against the CPU oracle's full
construction (oracle/host.build_descriptor, itself pinned to the reference's
descriptors in tests/test_oracle.py): tiny key sets, n = 1 and n = 64 leaves,
b = n, buckets past the shared-memory sort (> 16384 keys), rotate-cached
leaves above the cache threshold, and the query clamp of empty trailing
buckets.  Descriptor bytes and all query outputs must be identical."""

import numpy as np
import pytest

import oracle.host as OH
from paper_2308_09561_b200 import recsplit
from paper_2308_09561_b200.errors import DuplicateKeyError, InvalidParameterError
from paper_2308_09561_b200.keys import synthetic_hashed, synthetic_keys

pytestmark = pytest.mark.gpu

CASES = [
    # (N, b, n, mode, gen)
    (1, 1, 1, 1, 1),
    (2, 2, 1, 0, 2),
    (3, 8, 2, 1, 3),
    (5, 100, 4, 2, 4),
    (64, 64, 64, 0, 5),
    (64, 64, 64, 1, 6),
    (200, 200, 64, 1, 7),
    (1000, 16, 16, 0, 8),
    (1000, 1000, 1, 1, 9),
    (3000, 40, 40, 2, 10),
    (20000, 2000, 40, 2, 11),
    (40000, 20000, 30, 1, 12),   # buckets of ~20000 keys: the O(m^2) fallback sort
    (7777, 333, 24, 1, 13),
]


@pytest.mark.parametrize("N,b,n,mode,gen", CASES)
def test_build_matches_oracle(N, b, n, mode, gen):
    hi, lo = synthetic_hashed(N, gen)
    desc = recsplit.build_hashed(hi, lo, b, n, mode)
    blob = desc.serialize()
    ref_blob, res = OH.build_descriptor(hi, lo, b, n, mode)
    assert blob == ref_blob, (N, b, n, mode)
    out = desc.query_hashed_many(hi, lo)
    assert (out == OH.query(res, n, mode, 8, hi, lo)).all()
    assert (np.sort(out.astype(np.int64)) == np.arange(N)).all()
    assert recsplit.MphfDescriptor.deserialize(blob).serialize() == blob


def test_query_foreign_keys_match_oracle():
    """Keys outside the set still get the reference's (clamped) answers."""
    hi, lo = synthetic_hashed(5000, 21)
    desc = recsplit.build_hashed(hi, lo, 500, 24, 1)
    _, res = OH.build_descriptor(hi, lo, 500, 24, 1)
    qh, ql = synthetic_hashed(20000, 22)
    assert (desc.query_hashed_many(qh, ql) == OH.query(res, 24, 1, 8, qh, ql)).all()


def test_duplicates_and_parameters():
    keys = synthetic_keys(100, 3)
    with pytest.raises(DuplicateKeyError):
        recsplit.build(keys + [keys[17]], 50, 16)
    for b, n in ((10, 65), (10, 0), (5, 10)):
        with pytest.raises(InvalidParameterError):
            recsplit.build(keys, b, n)
    with pytest.raises(InvalidParameterError):
        recsplit.build([], 10, 4)


def test_duplicates_on_the_device_paths():
    """The asynchronous bucketize reports equal codes from run(): equal master
    codes -> HashCollisionError (build_hashed_device); a repeated key in a
    host blob -> DuplicateKeyError (build_blob, after the salt retry)."""
    import numpy as np

    from paper_2308_09561_b200 import device as dev
    from paper_2308_09561_b200.errors import HashCollisionError

    hi, lo = synthetic_hashed(3000, 23)
    hi[2999], lo[2999] = hi[5], lo[5]
    d_hi, d_lo = dev.DeviceBuffer.from_host(hi), dev.DeviceBuffer.from_host(lo)
    with pytest.raises(HashCollisionError):
        recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, 3000, 300, 20, 1)
    keys = np.arange(4000, dtype="<u8")
    keys[3999] = keys[123]
    blob = np.frombuffer(keys.tobytes(), dtype=np.uint8)
    with pytest.raises(DuplicateKeyError):
        recsplit.build_blob(blob, 8, 400, 20, 1)
    # and a clean build through the same path still matches the host path
    keys[3999] = 10**9
    blob = np.frombuffer(keys.tobytes(), dtype=np.uint8)
    assert recsplit.build_blob(blob, 8, 400, 20, 1).serialize() == recsplit.build(
        [k.tobytes() for k in keys], 400, 20, 1).serialize()


def test_large_build_is_a_bijection():
    """10x the C4 key count (N = 1e8): no 32-bit index overflows anywhere on
    the path; checked by size-independent properties (every key maps into
    [0, N) exactly once, on the device; the descriptor round-trips)."""
    from paper_2308_09561_b200 import device as dev

    N = 100_000_000
    hi, lo = synthetic_hashed(N, 2024)
    d_hi, d_lo = dev.DeviceBuffer.from_host(hi), dev.DeviceBuffer.from_host(lo)
    desc = recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, 2000, 40, 1)
    assert desc.n_keys == N
    ok, off = desc.device().verify(hi, lo)
    assert ok and off == -1
    blob = desc.serialize()
    assert recsplit.MphfDescriptor.deserialize(blob).serialize() == blob
    assert len(blob) * 8 / N < 1.7  # ~1.61 bits/key at n=40, b=2000


def _steal_search(hi, lo, off, max_seed=1 << 40):
    """The stealing kernel's path: device pointers, no counters requested."""
    from paper_2308_09561_b200 import device as dev
    from paper_2308_09561_b200._kernels import kernels as K

    L = len(off) - 1
    bufs = [dev.DeviceBuffer.from_host(np.ascontiguousarray(x, dtype=np.uint64)) for x in (hi, lo)]
    d_off = dev.DeviceBuffer.from_host(np.asarray(off, dtype=np.int64))
    d_s, d_f = dev.DeviceBuffer(8 * L), dev.DeviceBuffer(8 * L)
    try:
        K.leaf_search_device(bufs[0].ptr, bufs[1].ptr, d_off.ptr, L, 0, d_s.ptr, d_f.ptr, max_seed=max_seed)
        dev.sync()
        return d_s.download(np.int64, L), d_f.download(np.uint64, L)
    finally:
        for b_ in bufs + [d_off, d_s, d_f]:
            b_.free()


def test_steal_kernel_ragged_batch_matches_counting_kernel():
    """Ragged CSR leaves of 1..64 keys in one batch (n = 1 leaves, 32-bit and
    64-bit masks mixed): the stealing kernel's seeds and f bits equal the
    fixed-team kernel's (which also returns the reference's counters)."""
    from paper_2308_09561_b200._kernels import kernels as K

    rng = np.random.default_rng(77)
    sizes = np.concatenate([[1, 25, 64, 33, 2], rng.integers(1, 49, 600)])
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    hi, lo = synthetic_hashed(int(off[-1]), 4242)
    s_ref, f_ref, _ = K.leaf_search_batch(hi, lo, off, 0)
    s, f = _steal_search(hi, lo, off)
    assert (s == s_ref).all() and (f == f_ref).all()


def test_steal_kernel_exhaustion_and_single_leaf():
    """max_seed cuts: a leaf whose minimum seed is >= max_seed reports -1
    (the reference's exhaustion value, _core.pyx:223-229) and the others are
    unaffected; a lone leaf (all warps join it) gives the oracle's seed."""
    import oracle

    n = 40
    hi, lo = synthetic_hashed(8 * n, 99)
    off = np.arange(0, 9 * n, n)
    ref = [oracle.search_plain(hi[i * n : (i + 1) * n], lo[i * n : (i + 1) * n], n, 1 << 40)[0] for i in range(8)]
    cut = sorted(ref)[4]  # half of the leaves need more seeds than this
    s, f = _steal_search(hi, lo, off, max_seed=cut)
    assert s.tolist() == [x if x < cut else -1 for x in ref]
    assert all(int(f[i]) == 0 for i in range(8) if ref[i] >= cut)
    s1, f1 = _steal_search(hi[:n], lo[:n], np.array([0, n]))
    assert int(s1[0]) == ref[0]
    e = oracle.edges_plain(hi[:n], lo[:n], ref[0], n)
    assert int(f1[0]) == oracle.orient(e, n)


@pytest.mark.parametrize("n", [0, 1, 2, 255, 2047, 2048, 2049, 100_000, 1_482_000, 4096 * 2048 + 3])
def test_exclusive_scan_lengths(n):
    """The device scan every build stage uses (shk_exclusive_scan): one tile,
    tile edges, the per-tile carry loop and (past 4096 tiles) the recursive
    scan of the tile totals, against numpy's cumsum (recsplit.py:485)."""
    from paper_2308_09561_b200 import device as dev

    rng = np.random.default_rng(n + 1)
    a = rng.integers(0, 1 << 40, size=max(n, 1), dtype=np.int64)[:n]
    d_in = dev.DeviceBuffer.from_host(a if n else np.zeros(1, dtype=np.int64))
    d_out = dev.DeviceBuffer(8 * (n + 1))
    dev.exclusive_scan_device(d_in, d_out, n)
    got = d_out.download(np.int64, n + 1)
    want = np.concatenate([[0], np.cumsum(a)]).astype(np.int64)
    assert np.array_equal(got, want)
