"""GPU parity: every CUDA kernel against the reference's own outputs.

Fixtures under tests/golden/ were produced by running the REAL reference
(tests/golden/make_golden.py, compiled Cython backend).  Bit-exact equality
is required everywhere (integer/byte work): seeds, per-leaf counters, f bits,
split seeds and eval counts, ribbon rows and words, Rice decode, blake2b,
serialized descriptors and query outputs.
"""

import hashlib

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def sha(b):
    return hashlib.sha256(b).hexdigest()


def test_blake2b_vectors(K):
    g = golden("kat.json")["blake2b"]
    by_salt = {}
    for r in g:
        by_salt.setdefault(r["salt"], []).append(r)
    for salt, rows in by_salt.items():
        keys = [bytes.fromhex(r["key"]) for r in rows]
        hi, lo = K.blake2b128_many(keys, salt)
        assert [int(x) for x in hi] == [r["hi"] for r in rows]
        assert [int(x) for x in lo] == [r["lo"] for r in rows]


@pytest.mark.parametrize("key_len", [1, 3, 7, 8, 9, 15, 16, 17, 24, 31, 32, 33, 64, 100, 127, 128])
def test_blake2b_fixed_lengths(key_len):
    """Fixed-length fingerprint kernel (one specialisation per message-word
    count: <= 8, <= 16, <= 32, <= 128 bytes; word and byte loads) against the
    reference's definition, keys.py:39-58: hashlib.blake2b(key, digest_size=16,
    salt=pack("<QQ", salt, 0)) unpacked "<QQ" -> (hi, lo)."""
    import struct

    from paper_2308_09561_b200 import device as dev

    rng = np.random.default_rng(1000 + key_len)
    N = 777
    blob = rng.integers(0, 256, N * key_len, dtype=np.uint8)
    for salt in (0, 5, (1 << 64) - 1):
        hi, lo = dev.blake2b_fixed_host(blob, key_len, salt)
        raw = blob.tobytes()
        for i in range(N):
            d = hashlib.blake2b(raw[i * key_len : (i + 1) * key_len], digest_size=16,
                                salt=struct.pack("<QQ", salt, 0)).digest()
            eh, el = struct.unpack("<QQ", d)
            assert (int(hi[i]), int(lo[i])) == (eh, el), (key_len, salt, i)


@pytest.mark.parametrize("which", ["plain", "rotate", "rotate_cached"])
def test_leaf_search_golden(K, which):
    recs = golden("leaves.json")
    for r in recs:
        n = r["n"]
        exp = r[which]
        if which == "plain":
            (t, fb) = K.search_plain_fbits(r["hi"], r["lo"], n, 1 << 40)
        else:
            ck = 0 if which == "rotate" else exp["ck"]
            (t, fb) = K.search_rotate_fbits(r["hi"], r["lo"], n, ck, 1 << 40)
        assert list(t) == exp["stats"], (which, n, r["gen"])
        assert fb == exp["fbits"], (which, n, r["gen"])


def test_leaf_search_batched_mixed_sizes(K):
    """All golden leaves of all sizes in ONE launch (CSR), per mode."""
    recs = golden("leaves.json")
    hi = np.concatenate([np.asarray(r["hi"], dtype=np.uint64) for r in recs])
    lo = np.concatenate([np.asarray(r["lo"], dtype=np.uint64) for r in recs])
    off = np.cumsum([0] + [r["n"] for r in recs])
    for mode, key in ((0, "plain"), (1, "rotate")):
        seeds, fb, st = K.leaf_search_batch(hi, lo, off, mode)
        assert [int(s) for s in seeds] == [r[key]["seed"] for r in recs]
        assert [int(f) for f in fb] == [r[key]["fbits"] for r in recs]
        assert st.tolist() == [r[key]["stats"][1:] for r in recs]
    # rotate-cached with recsplit's rule (cache only above 32 keys)
    seeds, fb, st = K.leaf_search_batch(hi, lo, off, 1, 8, 32)
    assert [int(s) for s in seeds] == [r["rotate_cached"]["seed"] for r in recs]
    assert [int(f) for f in fb] == [r["rotate_cached"]["fbits"] for r in recs]


@pytest.mark.parametrize("team", [1, 2, 4, 8])
def test_leaf_team_sizes_agree(K, team):
    recs = [r for r in golden("leaves.json") if r["n"] >= 2]
    hi = np.concatenate([np.asarray(r["hi"], dtype=np.uint64) for r in recs])
    lo = np.concatenate([np.asarray(r["lo"], dtype=np.uint64) for r in recs])
    off = np.cumsum([0] + [r["n"] for r in recs])
    for mode, key in ((0, "plain"), (1, "rotate")):
        seeds, fb, st = K.leaf_search_batch(hi, lo, off, mode, team_warps=team)
        assert [int(s) for s in seeds] == [r[key]["seed"] for r in recs]
        assert st.tolist() == [r[key]["stats"][1:] for r in recs]


def test_leaf_max_seed_cutoff(K):
    # reference KAT (test_shockhash.py:137-141): hashed_leaf(8, 0) has minimum
    # plain seed 2, so a cutoff of 1 fails and 3 succeeds
    from conftest import hashed_leaf

    keys = hashed_leaf(8, 0)
    hi = [k.hi for k in keys]
    lo = [k.lo for k in keys]
    t = K.search_plain(hi, lo, 8, 1)
    assert t[0] == -1 and t[1] == 8
    assert K.search_plain(hi, lo, 8, 3)[0] == 2
    assert K.search_plain(hi, lo, 8, 1 << 40)[0] == 2


@pytest.mark.parametrize("cfg,sample", [(1, None), (3, 2000), (5, None)])
def test_leaf_config_golden(K, cfg, sample):
    from paper_2308_09561_b200 import workloads as W

    g = golden(f"c{cfg}.json")
    hi, lo = W.leaf_inputs(cfg, g["leaves"])
    n = g["n"]
    assert [int(x) for x in hi[0]] == g["hi0"]
    off = np.arange(0, n * (g["leaves"] + 1), n)
    seeds, fb, st = K.leaf_search_batch(hi, lo, off, 0)
    assert [int(s) for s in seeds] == g["seeds"]
    assert [int(f) for f in fb] == g["fbits"]
    assert st[:, :3].tolist() == g["stats"]
    if cfg == 1:
        assert sha(seeds.astype("<i8").tobytes() + fb.astype("<u8").tobytes())[:16] == g["sha16"]


@pytest.mark.parametrize("cfg", [3, 5])
def test_leaf_config_full_population(K, cfg):
    """Every leaf of C3 (100,000 x n=32) and C5 (20,000 x n=56) against the
    reference's own minimum seed, f bits and filter-pass counter."""
    import os

    from conftest import GOLDEN, full_leaf_golden
    from paper_2308_09561_b200 import workloads as W

    if not os.path.exists(os.path.join(GOLDEN, f"c{cfg}_full.json")):
        pytest.skip(f"c{cfg}_full golden not generated")
    gs, gf, gp, meta = full_leaf_golden(cfg)
    hi, lo = W.leaf_inputs(cfg)
    n = meta["n"]
    off = np.arange(0, n * (meta["leaves"] + 1), n)
    seeds, fb, st = K.leaf_search_batch(hi, lo, off, 0)
    bad = np.flatnonzero(seeds != gs)
    assert bad.size == 0, (bad[:10], seeds[bad[:10]], gs[bad[:10]])
    assert (fb == gf).all(), np.flatnonzero(fb != gf)[:10]
    assert (st[:, 0] == (gs + 1) * n).all()
    assert (st[:, 1].astype(np.uint64) == gp).all() and (st[:, 2] == st[:, 1]).all()
    assert sha(seeds.astype("<i8").tobytes() + fb.astype("<u8").tobytes())[:16] == meta["sha16"]


@pytest.mark.parametrize("cfg", [3, 5])
def test_leaf_config_full_population_device(K, cfg):
    """The bench path (device pointers, no stats) on every leaf of C3 / C5."""
    import os

    from conftest import GOLDEN, full_leaf_golden
    from paper_2308_09561_b200 import device as dev
    from paper_2308_09561_b200 import workloads as W

    if not os.path.exists(os.path.join(GOLDEN, f"c{cfg}_full.json")):
        pytest.skip(f"c{cfg}_full golden not generated")
    gs, gf, _, meta = full_leaf_golden(cfg)
    hi, lo = W.leaf_inputs(cfg)
    L, n = meta["leaves"], meta["n"]
    bufs = [dev.DeviceBuffer.from_host(np.ascontiguousarray(x).ravel()) for x in (hi, lo)]
    d_off = dev.DeviceBuffer.from_host(np.arange(0, (L + 1) * n, n, dtype=np.int64))
    d_seed, d_fb = dev.DeviceBuffer(8 * L), dev.DeviceBuffer(8 * L)
    try:
        K.leaf_search_device(bufs[0].ptr, bufs[1].ptr, d_off.ptr, L, 0, d_seed.ptr, d_fb.ptr)
        dev.sync()
        assert (d_seed.download(np.int64, L) == gs).all()
        assert (d_fb.download(np.uint64, L) == gf).all()
    finally:
        for b_ in bufs + [d_off, d_seed, d_fb]:
            b_.free()


def test_split_search_golden(K):
    from paper_2308_09561_b200.keys import synthetic_hashed

    for r in golden("split.json")["cases"]:
        hi, lo = synthetic_hashed(r["m"], r["gen"])
        seed, evals = K.split_seed_search(hi, lo, r["sizes"], 1 << 30)
        assert (seed, evals) == (r["seed"], r["evals"]), r
        parts = K.split_parts(hi, lo, seed, r["sizes"])
        assert sha(np.asarray(parts, "<i8").tobytes()) == r["parts_sha"]


def test_ribbon_golden(K):
    from paper_2308_09561_b200.keys import synthetic_hashed

    for r in golden("ribbon.json"):
        N, m, seed = r["N"], r["m"], r["seed"]
        rng = np.random.default_rng(N)
        hi, lo = synthetic_hashed(N, r["gen"])
        rhs = rng.integers(0, 2, N).astype(np.uint8)
        st, p0, p1 = K.ribbon_rows(hi, lo, seed, m)
        assert sha(np.asarray(st, "<i8").tobytes() + np.asarray(p0, "<u8").tobytes() + np.asarray(p1, "<u8").tobytes()) == r["rows_sha"]
        w = K.ribbon_solve(st, p0, p1, rhs, m)
        assert (w is not None) == r["solvable"]
        if w is not None:
            assert sha(np.asarray(w, "<u8").tobytes()) == r["words_sha"]
            if r["words"] is not None:
                assert [int(x) for x in w] == r["words"]
            q = K.ribbon_query_many(st, p0, p1, w, m)
            assert (q == rhs).all()


def test_ribbon_order_independence(K):
    """any row order gives the same words."""
    from paper_2308_09561_b200.keys import synthetic_hashed

    N = 50_000
    hi, lo = synthetic_hashed(N, 77)
    rhs = (hi >> np.uint64(7) & np.uint64(1)).astype(np.uint8)
    m = max(128, int(np.ceil(1.05 * N)))
    st, p0, p1 = K.ribbon_rows(hi, lo, 0, m)
    w = K.ribbon_solve(st, p0, p1, rhs, m)
    perm = np.random.default_rng(0).permutation(N)
    w2 = K.ribbon_solve(st[perm], p0[perm], p1[perm], rhs[perm], m)
    assert w is not None and (w == w2).all()


def test_rice_decode_golden(K):
    g = golden("rice.json")
    words = np.asarray(g["words"], dtype=np.uint64)
    vals, poss = K.rice_decode_many(words, g["bit_len"], 0, [gg for _, gg in g["items"]])
    assert [int(v) for v in vals] == [v for v, _ in g["items"]]
    assert int(poss[-1]) == g["bit_len"]


def test_rice_truncation_raises(K):
    from paper_2308_09561_b200 import errors, recsplit

    w = recsplit.BitWriter()
    w.rice(1000, 0)
    with pytest.raises(errors.FormatError):
        recsplit.rice_decode(w.to_array(), w.bit_len - 5, 0, 0)


def test_c2_build_golden():
    """C2: N=1e5, n=24, b=500, rotate -> identical descriptor and 1e6 queries."""
    from paper_2308_09561_b200 import recsplit
    from paper_2308_09561_b200 import workloads as W

    g = golden("c2.json")
    keys = W.keys_as_bytes(W.build_keys(2))
    desc = recsplit.build(keys, 500, 24)
    blob = desc.serialize()
    with open("tests/golden/c2_desc.bin", "rb") as f:
        ref = f.read()
    assert len(blob) == len(ref)
    assert blob == ref
    assert sha(blob) == g["desc_sha"]
    hi, lo = W.blake2b_host(keys, 0)
    idx = W.query_indices(2)
    out = desc.query_hashed_many(hi[idx], lo[idx])
    assert sha(np.asarray(out, "<u8").tobytes()) == g["query_sha"]
    own = desc.query_hashed_many(hi, lo)
    assert (np.bincount(own.astype(np.int64), minlength=len(keys)) == 1).all()
    # query_many(keys) end to end (the pipelined host-blob path, chunks of 4M
    # keys: 1e6 queries are one chunk, so also a 9M-query batch of the same keys)
    qkeys = [keys[i] for i in idx]
    assert sha(np.asarray(desc.query_many(qkeys), "<u8").tobytes()) == g["query_sha"]
    blob9 = np.frombuffer(b"".join(qkeys) * 9, dtype=np.uint8)
    out9 = desc.query_blob(blob9, 8)
    assert (out9.reshape(9, -1) == np.asarray(out, dtype=np.uint64)[None, :]).all()


@pytest.mark.parametrize("env", [
    {"SHK_TREE_SLOT_AWARE": "0"},          # every warp slot takes split nodes
    {"SHK_TREE_SLOW_WID": "4"},            # splits on the 4 lowest slots only
    {"SHK_TREE_SLOW_WID": "31", "SHK_TREE_IDLE_WID": "24"},
    {"SHK_TREE_HANDOFF_TW": "0"},          # no tail hand-off
    {"SHK_TREE_HANDOFF_TW": "1"},          # resume teams of 1, 2, 4 warps
    {"SHK_TREE_HANDOFF_TW": "2"},
    {"SHK_TREE_HANDOFF_TW": "4"},
])
def test_c2_build_schedule_independent(monkeypatch, env):
    """The persistent tree kernel's schedule (which warp slots take split nodes
    and which take leaves, shk_tree.cu) changes only the order of the work:
    the C2 descriptor is the reference's bytes under every schedule."""
    from paper_2308_09561_b200 import recsplit
    from paper_2308_09561_b200 import workloads as W

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    keys = W.keys_as_bytes(W.build_keys(2))
    blob = recsplit.build(keys, 500, 24).serialize()
    assert sha(blob) == golden("c2.json")["desc_sha"]


@pytest.mark.parametrize("n,mode", [(24, 1), (40, 2)])
def test_tree_handoff_exact(monkeypatch, n, mode):
    """Tail hand-off (shk_tree.cu): once every leaf is handed out, the
    leaves still searching stop at a round boundary and tree_resume_kernel
    finishes them with multi-warp teams.  The seeds (Rice stream), the choice
    bits and every reference counter equal the uninterrupted search's, for the
    plain rotation and the k-aligned cached rotation."""
    from paper_2308_09561_b200 import recsplit
    from paper_2308_09561_b200 import shockhash as leaf_mod
    from paper_2308_09561_b200 import workloads as W
    from paper_2308_09561_b200.keys import master_hash_many
    from paper_2308_09561_b200._kernels import kernels as K

    keys = W.keys_as_bytes(W.build_keys(2))
    hi, lo = master_hash_many(keys, 0)
    N, b = len(keys), 500
    nb = (N + b - 1) // b
    ck = leaf_mod.DEFAULT_CACHE_K if mode == 2 else 0
    out = {}
    for tw in ("0", "8", "2"):
        monkeypatch.setenv("SHK_TREE_HANDOFF_TW", tw)
        gb = K.GpuBuild(hi, lo, nb)
        plans = recsplit.packed_plans_for_prefix(gb.key_prefix(), n, recsplit.leaf_g_table(n))
        st = gb.run(plans, 1, ck, leaf_mod.CACHE_MIN_LEAF, 0, nb, leaf_mod.MAX_SEED)
        words, bits, _ = gb.stream()
        out[tw] = (st, words, bits, gb.choice())
        gb.close()
    assert out["0"][0][7] == 0
    for tw in ("8", "2"):
        st, words, bits, ch = out[tw]
        assert st[7] > 0, "no leaf was handed off"
        assert (st[:7] == out["0"][0][:7]).all()
        assert bits == out["0"][2] and (words == out["0"][1]).all()
        assert (ch == out["0"][3]).all()


def test_small_builds_golden():
    from paper_2308_09561_b200 import recsplit
    from paper_2308_09561_b200.keys import synthetic_hashed, synthetic_keys

    for r in golden("builds.json"):
        if r.get("hashed"):
            hi, lo = synthetic_hashed(r["N"], r["gen"])
            desc = recsplit.build_hashed(hi, lo, r["b"], r["n"], r["mode"])
            assert sha(desc.serialize()) == r["desc_sha"]
            assert sha(np.asarray(desc.query_hashed_many(hi, lo), "<u8").tobytes()) == r["query_sha"]
            continue
        keys = synthetic_keys(r["N"], r["gen"])
        desc = recsplit.build(keys, r["b"], r["n"], r["mode"])
        blob = desc.serialize()
        if r["desc_hex"] is not None:
            assert blob.hex() == r["desc_hex"], r
        assert sha(blob) == r["desc_sha"], r
        assert sha(np.asarray(desc.query_many(keys), "<u8").tobytes()) == r["query_sha"], r


def _synthetic_hashed(count, gen_seed):
    from paper_2308_09561_b200.keys import synthetic_hashed

    return synthetic_hashed(count, gen_seed)


def test_search_bruteforce_golden(K):
    for r in golden("experiments.json")["bruteforce"]:
        hi, lo = _synthetic_hashed(r["n"], r["gen"])
        assert K.search_bruteforce(hi, lo, r["n"], r["max_seed"]) == (r["seed"], r["evals"]), r


def test_search_bruteforce_vs_oracle(K):
    """Larger n than the fixtures, several doubling batches deep."""
    import oracle

    for n, gen in ((17, 5), (18, 6)):
        hi, lo = _synthetic_hashed(n, gen)
        assert K.search_bruteforce(hi, lo, n, 1 << 40) == oracle.search_bruteforce(hi, lo, n, 1 << 40)


def test_mc_filter_golden(K):
    for r in golden("experiments.json")["mc_filter"]:
        assert K.mc_filter_pass_count(r["n"], r["trials"], r["entropy"]) == r["passes"], r


def test_enumerate_outcomes_golden(K):
    for r in golden("experiments.json")["enumerate"]:
        assert K.enumerate_outcomes(r["n"]) == (r["pf_count"], r["sum_2c"]), r
    assert K.enumerate_outcomes(0) == (1, 1)
    with pytest.raises(ValueError):
        K.enumerate_outcomes(9)


@pytest.mark.parametrize("n", [7, 8])
def test_enumerate_outcomes_closed_form(K, n):
    """n = 7, 8 ((n^2)^n = 6.8e11 / 2.8e14 tuples) are out of the oracle's
    reach; they are checked against the closed-form census in
    tests/enum_census.py, which is itself pinned to the reference's n <= 6
    outputs by tests/test_oracle.py."""
    from enum_census import census

    assert K.enumerate_outcomes(n) == (census(n, 1), census(n, 2))
