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
