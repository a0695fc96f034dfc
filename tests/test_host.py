"""CPU tests of the host side: the C-ABI library loads and exports every
symbol of include/shockhash_b200.h, the scalar hash API, plans and Rice
parameters, the byte format, pseudoforest utilities, error mapping, and the
fail-loudly contract without a GPU."""

import hashlib
import itertools
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden


def header_symbols():
    src = open(os.path.join(ROOT, "include", "shockhash_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(shk_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    import ctypes

    from paper_2308_09561_b200._kernels import _lib

    lib = _lib.load_library()
    syms = header_symbols()
    assert len(syms) >= 40
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.EXPORTED, f"{s} has no ctypes signature"
    # and the .so carries sm_100a code
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_lib.LIB_PATH} 2>/dev/null").read()
    if out:
        assert "sm_100a" in out


def test_scalar_api_matches_reference(K):
    g = golden("kat.json")
    for r in g["scalars"]:
        assert K.mix64(r["hi"]) == r["mix64"]
        assert K.seed_mixer(r["s"], r["tag"]) == r["seed_mixer"]
        assert K.remix(r["hi"], r["lo"], r["s"], r["tag"]) == r["remix"]
        assert K.hash_range(r["hi"], r["n"]) == r["hash_range"]
        assert list(K.leaf_pair(r["hi"], r["lo"], r["s"], r["n"])) == r["leaf_pair"]
        assert K.split_bit(r["hi"], r["lo"], r["s"]) == r["split_bit"]
    for r in g["leaf_cell"]:
        assert K.leaf_cell(r["hi"], r["lo"], r["q"], r["n"], r["mode"], r["ck"], r["choice"]) == r["cell"]
    assert K.mix64(0x9E3779B97F4A7C15) == 0xE220A8397B1DCDAF


def test_batch_mixers_match_scalar(K):
    rng = np.random.default_rng(2)
    h = rng.integers(0, 2**63, 300).astype(np.uint64)
    l = rng.integers(0, 2**63, 300).astype(np.uint64)
    rb = K.remix_batch(h, l, 9, 4)
    assert all(int(rb[i]) == K.remix(int(h[i]), int(l[i]), 9, 4) for i in range(0, 300, 37))
    hr = K.hash_range_batch(h, 37)
    assert all(int(hr[i]) == K.hash_range(int(h[i]), 37) for i in range(0, 300, 41))


def test_compute_fails_loudly_without_gpu(K):
    from paper_2308_09561_b200._kernels import _lib

    if _lib.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.BackendUnavailableError):
        K.search_plain([1, 2], [3, 4], 2, 100)
    with pytest.raises(_lib.BackendUnavailableError):
        from paper_2308_09561_b200 import recsplit

        recsplit.build_hashed(np.arange(100, dtype=np.uint64), np.arange(100, dtype=np.uint64), 50, 16)


def test_get_backend_single():
    from paper_2308_09561_b200._kernels import BACKEND_NAME, get_backend

    assert BACKEND_NAME == "cuda"
    assert get_backend() is get_backend("compiled")
    with pytest.raises(ValueError):
        get_backend("pure")


def test_plan_shapes():
    from paper_2308_09561_b200.recsplit import plan

    # test_recsplit.py:16-36 KATs
    assert plan(0, 30) == ("leaf", 0)
    assert plan(30, 30) == ("leaf", 30)
    assert plan(120, 30) == ("split", (30, 30, 30, 30))
    assert plan(100, 30) == ("split", (30, 30, 30, 10))
    assert plan(360, 30) == ("split", (120, 120, 120))
    k, s = plan(2000, 30)
    assert k == "split" and len(s) == 2 and s[0] % 360 == 0
    k, s = plan(100, 16)
    assert s[0] % 16 == 0 and sum(s) == 100
    # C4 tree: 2000 -> (1440, 560)
    assert plan(2000, 40) == ("split", (1440, 560))


def test_plan_invariants_random():
    from paper_2308_09561_b200.recsplit import plan

    rng = np.random.default_rng(0)
    for _ in range(2000):
        m, n = int(rng.integers(0, 5000)), int(rng.integers(1, 65))
        k, a = plan(m, n)
        if k == "leaf":
            assert m <= n and a == m
        else:
            assert sum(a) == m and all(1 <= x < m for x in a) and len(a) <= 4


def test_flatten_plan_matches_reference_tables():
    import json

    from paper_2308_09561_b200.recsplit import flatten_plan

    plans = {}
    for n in (8, 16, 20, 24, 30, 40, 56, 64):
        for m in list(range(0, 200)) + list(range(400, 2600, 37)):
            plans[f"{m},{n}"] = [list(x) for x in flatten_plan(m, n, np.arange(65))] if m > 0 else None
    got = hashlib.sha256(json.dumps(plans, sort_keys=True, default=int).encode()).hexdigest()
    assert got == golden("split.json")["plans_sha"]


def test_rice_params_match_reference():
    from paper_2308_09561_b200.recsplit import leaf_rice_param, plan, split_rice_param

    g = golden("split.json")
    assert [leaf_rice_param(m) for m in range(65)] == g["leaf_g"]
    for r in g["cases"]:
        assert split_rice_param(r["m"], tuple(r["sizes"])) == r["g"]
        assert tuple(plan(r["m"], r["n"])[1]) == tuple(r["sizes"])


def test_bitwriter_rice_kats():
    from paper_2308_09561_b200 import errors, recsplit

    w = recsplit.BitWriter()
    w.rice(0, 0)
    assert w.bit_len == 1 and int(w.to_array()[0]) & 1 == 0
    w2 = recsplit.BitWriter()
    w2.rice(5, 2)
    assert w2.bit_len == 4 and int(w2.to_array()[0]) & 0xF == 0b0101
    g = golden("rice.json")
    w3 = recsplit.BitWriter()
    for v, gg in g["items"]:
        w3.rice(v, gg)
    assert w3.bit_len == g["bit_len"] and [int(x) for x in w3.to_array()] == g["words"]
    with pytest.raises(errors.InvalidParameterError):
        w.append(4, 2)
    with pytest.raises(errors.InvalidParameterError):
        w.rice(-1, 0)


def _desc_from_oracle_bytes():
    from paper_2308_09561_b200 import recsplit

    with open(os.path.join(ROOT, "tests", "golden", "c2_desc.bin"), "rb") as f:
        blob = f.read()
    return blob, recsplit.MphfDescriptor.deserialize(blob)


def test_descriptor_roundtrip_bytes():
    blob, d = _desc_from_oracle_bytes()
    assert d.serialize() == blob
    st = d.stats()
    assert st["seed_stream_bits"] + st["bucket_offset_bits"] + st["retrieval_bits"] + st["header_bits"] == st["total_bits"]
    assert abs(st["bits_per_key"] - 1.81024) < 1e-9  # SURVEY.md App. B anchor
    assert d.offset_width == 32 and d.nbuckets == 200


def test_descriptor_rejects_corruption():
    from paper_2308_09561_b200 import errors, recsplit

    blob, _ = _desc_from_oracle_bytes()
    for bad in (b"XXXX" + blob[4:], blob[:30], blob + b"\x00", blob[:-8]):
        with pytest.raises(errors.FormatError):
            recsplit.MphfDescriptor.deserialize(bad)
    b2 = bytearray(blob)
    b2[4] = 99
    with pytest.raises(errors.FormatError):
        recsplit.MphfDescriptor.deserialize(bytes(b2))


def test_pseudoforest_utilities_exhaustive():
    from paper_2308_09561_b200 import pseudoforest as pf
    from paper_2308_09561_b200.errors import ContractViolationError, InvalidParameterError

    for n in (1, 2, 3, 4):
        for cells in itertools.product(range(n), repeat=2 * n):
            edges = [(cells[2 * i], cells[2 * i + 1]) for i in range(n)]
            assert pf.is_pseudoforest(edges, n) == (pf.count_orientations(edges, n) > 0)
    uf = pf.UnionFindPF(2)
    assert uf.try_insert_edge(0, 1) and uf.try_insert_edge(0, 1)
    assert not uf.try_insert_edge(0, 1) and uf.poisoned
    with pytest.raises(ContractViolationError):
        uf.try_insert_edge(0, 1)
    with pytest.raises(InvalidParameterError):
        pf.is_pseudoforest([(0, 3)], 3)
    assert pf.count_orientations([(0, 1), (1, 2), (2, 0), (3, 4), (4, 3)], 5) == 4


def test_parameter_validation_before_device():
    from paper_2308_09561_b200 import errors, recsplit
    from paper_2308_09561_b200 import shockhash as sh
    from paper_2308_09561_b200.keys import HashedKey

    keys = [HashedKey(i, i + 1) for i in range(4)]
    with pytest.raises(errors.UnsupportedLeafSizeError):
        sh.search_plain(keys, 65)
    with pytest.raises(errors.InvalidParameterError):
        sh.search_plain(keys, 5)
    with pytest.raises(errors.InvalidParameterError):
        sh.search_rotate_cached(keys, 4, k=0)
    with pytest.raises(errors.InvalidParameterError):
        sh.search(keys, 4, mode=9)
    with pytest.raises(errors.InvalidParameterError):
        recsplit.build([], 100, 16)
    with pytest.raises(errors.InvalidParameterError):
        recsplit.build([b"a"], 100, 65)
    with pytest.raises(errors.InvalidParameterError):
        recsplit.build([b"a"], 8, 16)
    with pytest.raises(errors.InvalidParameterError):
        recsplit.build([b"a"], 100, 16, mode=7)


def test_status_codes_map_to_reference_errors():
    from paper_2308_09561_b200 import errors
    from paper_2308_09561_b200._kernels import _lib

    for rc, exc in ((1, errors.ConstructionFailureError), (2, errors.FormatError), (3, errors.InvalidParameterError),
                    (4, errors.ConstructionFailureError)):
        with pytest.raises(exc):
            _lib.check(rc)
    with pytest.raises(_lib.BackendUnavailableError):
        _lib.check(-1001)
