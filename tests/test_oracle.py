"""Pin the CPU oracle (oracle/shk_oracle.c) against the reference's golden
vectors.  CPU only; these make the oracle a trustworthy checker for the
GPU parity tests."""

import hashlib
import os

import numpy as np
import pytest

import oracle
import oracle.host as OH
from conftest import ROOT, golden


def sha(b):
    return hashlib.sha256(b).hexdigest()


def synthetic_hashed(count, gen_seed):
    # keys.py:102-112 recipe (test input generator)
    base = np.uint64(OH._mix64_np(np.asarray([gen_seed], dtype=np.uint64))[0] ^ np.uint64(0x5851F42D4C957F2D))
    idx = np.arange(count, dtype=np.uint64)
    return OH._mix64_np(base + np.uint64(2) * idx), OH._mix64_np(base + np.uint64(2) * idx + np.uint64(1))


def test_mix64_kat():
    # test_keys.py:33-39 (SplitMix64 reference sequence)
    assert oracle.mix64(0x9E3779B97F4A7C15) == 0xE220A8397B1DCDAF
    assert oracle.mix64((2 * 0x9E3779B97F4A7C15) % 2**64) == 0x6E789E6AA1B965F4
    assert oracle.mix64((3 * 0x9E3779B97F4A7C15) % 2**64) == 0x06C45D188009454F


def test_scalar_golden():
    g = golden("kat.json")
    for r in g["scalars"]:
        assert oracle.mix64(r["hi"]) == r["mix64"]
        assert oracle.seed_mixer(r["s"], r["tag"]) == r["seed_mixer"]
        assert oracle.remix(r["hi"], r["lo"], r["s"], r["tag"]) == r["remix"]
        assert oracle.hash_range(r["hi"], r["n"]) == r["hash_range"]
        assert list(oracle.leaf_pair(r["hi"], r["lo"], r["s"], r["n"])) == r["leaf_pair"]
        assert oracle.split_bit(r["hi"], r["lo"], r["s"]) == r["split_bit"]
    for r in g["leaf_cell"]:
        assert oracle.leaf_cell(r["hi"], r["lo"], r["q"], r["n"], r["mode"], r["ck"], r["choice"]) == r["cell"]


@pytest.mark.parametrize("which", ["plain", "rotate", "rotate_cached"])
def test_leaf_golden(which):
    for r in golden("leaves.json"):
        n, e = r["n"], r[which]
        if which == "plain":
            t = oracle.search_plain(r["hi"], r["lo"], n, 1 << 40)
            edges = oracle.edges_plain(r["hi"], r["lo"], t[0], n)
        else:
            ck = 0 if which == "rotate" else e["ck"]
            t = oracle.search_rotate(r["hi"], r["lo"], n, ck, 1 << 40)
            edges = oracle.edges_rotate(r["hi"], r["lo"], t[0], n, ck)
        assert list(t) == e["stats"]
        assert oracle.orient(edges, n) == e["fbits"]


def test_c1_golden():
    from paper_2308_09561_b200 import workloads as W

    g = golden("c1.json")
    hi, lo = W.leaf_inputs(1)
    seeds = oracle.search_plain_batch(hi, lo)
    assert int(seeds.sum()) == g["sum_seed"] == 64870  # SURVEY.md App. B anchor
    assert seeds.tolist() == g["seeds"]
    fb = [oracle.orient(oracle.edges_plain(hi[i], lo[i], int(seeds[i]), 16), 16) for i in range(len(seeds))]
    assert fb == g["fbits"]
    assert sha(seeds.astype("<i8").tobytes() + np.asarray(fb, dtype="<u8").tobytes())[:16] == g["sha16"]


def test_c3_sample_golden():
    from paper_2308_09561_b200 import workloads as W

    g = golden("c3.json")
    hi, lo = W.leaf_inputs(3, 500)
    seeds = oracle.search_plain_batch(hi, lo)
    assert seeds.tolist() == g["seeds"][:500]


def test_c5_sample_golden():
    g = golden("c5.json")
    rng = np.random.default_rng(5)
    fp = rng.integers(0, 2**64, (20000, 56, 2), dtype=np.uint64)[:4]
    seeds = oracle.search_plain_batch(np.ascontiguousarray(fp[..., 0]), np.ascontiguousarray(fp[..., 1]))
    assert seeds.tolist() == g["seeds"][:4]


@pytest.mark.parametrize("cfg,count", [(3, 400), (5, 6)])
def test_full_population_golden_sample(cfg, count):
    """The C oracle on a sample of the full-population reference goldens
    (tests/golden/c{3,5}_full.bin): random C3 leaves, and the C5 leaves with
    the smallest seeds (so the CPU search stays short)."""
    from conftest import full_leaf_golden
    from paper_2308_09561_b200 import workloads as W

    gs, gf, gp, meta = full_leaf_golden(cfg)
    n = meta["n"]
    if cfg == 3:
        idx = np.sort(np.random.default_rng(33).choice(meta["leaves"], count, replace=False))
    else:
        idx = np.sort(np.argsort(gs, kind="stable")[:count])
    hi, lo = W.leaf_inputs(cfg)
    for i in idx:
        t = oracle.search_plain(hi[i], lo[i], n, 1 << 40)
        assert t[0] == int(gs[i]) and t[2] == int(gp[i]), (cfg, int(i))
        assert oracle.orient(oracle.edges_plain(hi[i], lo[i], t[0], n), n) == int(gf[i])
    assert int((gs + 1).sum()) == meta["seeds_tested"]


def test_split_golden():
    for r in golden("split.json")["cases"]:
        hi, lo = synthetic_hashed(r["m"], r["gen"])
        assert oracle.split_seed_search(hi, lo, r["sizes"], 1 << 30) == (r["seed"], r["evals"])
        parts = oracle.split_parts(hi, lo, r["seed"], r["sizes"])
        assert sha(parts.astype("<i8").tobytes()) == r["parts_sha"]
        assert OH.split_rice_param(r["m"], tuple(r["sizes"])) == r["g"]
    assert [OH.leaf_rice_param(m) for m in range(65)] == golden("split.json")["leaf_g"]


def test_ribbon_golden():
    for r in golden("ribbon.json"):
        N, m, seed = r["N"], r["m"], r["seed"]
        rng = np.random.default_rng(N)
        hi, lo = synthetic_hashed(N, r["gen"])
        rhs = rng.integers(0, 2, N).astype(np.uint8)
        st, p0, p1 = oracle.ribbon_rows(hi, lo, seed, m)
        assert sha(st.astype("<i8").tobytes() + p0.astype("<u8").tobytes() + p1.astype("<u8").tobytes()) == r["rows_sha"]
        w = oracle.ribbon_solve(st, p0, p1, rhs, m)
        assert (w is not None) == r["solvable"]
        if w is not None:
            assert sha(w.astype("<u8").tobytes()) == r["words_sha"]
            assert (oracle.ribbon_query(st, p0, p1, w, m) == rhs).all()


def test_rice_golden():
    g = golden("rice.json")
    pos = 0
    for v, gg in g["items"]:
        x, pos = oracle.rice_decode(g["words"], g["bit_len"], pos, gg)
        assert x == v
    assert pos == g["bit_len"]


def test_c2_full_build_golden():
    """C2 end to end on the oracle: identical descriptor bytes and 1e6 queries."""
    from paper_2308_09561_b200 import workloads as W

    g = golden("c2.json")
    keys = W.keys_as_bytes(W.build_keys(2))
    hi, lo = W.blake2b_host(keys, 0)
    blob, res = OH.build_descriptor(hi, lo, 500, 24)
    assert sha(blob) == g["desc_sha"]
    with open("tests/golden/c2_desc.bin", "rb") as f:
        assert blob == f.read()
    idx = W.query_indices(2)
    out = OH.query(res, 24, 1, 8, hi[idx], lo[idx])
    assert sha(out.astype("<u8").tobytes()) == g["query_sha"]


def test_small_builds_golden():
    from paper_2308_09561_b200 import workloads as W
    from paper_2308_09561_b200.keys import synthetic_keys

    for r in golden("builds.json"):
        if r.get("hashed"):
            hi, lo = synthetic_hashed(r["N"], r["gen"])
        else:
            hi, lo = W.blake2b_host(synthetic_keys(r["N"], r["gen"]), 0)
        blob, res = OH.build_descriptor(hi, lo, r["b"], r["n"], r["mode"])
        assert sha(blob) == r["desc_sha"], r
        out = OH.query(res, r["n"], r["mode"], 8, hi, lo)
        assert sha(out.astype("<u8").tobytes()) == r["query_sha"], r


def test_experiments_golden():
    """search_bruteforce / mc_filter_pass_count / enumerate_outcomes
    (_core.pyx:337-371, 778-860) against the reference's outputs."""
    g = golden("experiments.json")
    for r in g["bruteforce"]:
        hi, lo = synthetic_hashed(r["n"], r["gen"])
        assert oracle.search_bruteforce(hi, lo, r["n"], r["max_seed"]) == (r["seed"], r["evals"]), r
    for r in g["enumerate"]:
        if r["n"] <= 5:
            assert oracle.enumerate_outcomes(r["n"]) == (r["pf_count"], r["sum_2c"]), r
    for r in g["mc_filter"]:
        if r["n"] * r["trials"] <= 5_000_000:
            assert oracle.mc_filter_pass_count(r["n"], r["trials"], r["entropy"]) == r["passes"], r


def test_enumeration_census_pinned():
    """The closed form used for the GPU check at n = 7, 8 reproduces the
    reference's enumerate_outcomes for every n it was run at."""
    from enum_census import census

    for r in golden("experiments.json")["enumerate"]:
        assert (census(r["n"], 1), census(r["n"], 2)) == (r["pf_count"], r["sum_2c"])
    assert census(0, 1) == 1 and census(0, 2) == 1


def test_refbuild_matches_stock_reference():
    """The reference CPU arm (oracle/refbuild.py: the reference's compiled
    kernels under a restated build loop with a process pool) produces the
    STOCK reference's descriptor bytes: pinned on the first 100,000 C4 keys
    (b=2000, n=40, rotate) against shockhash.build from the unmodified
    package installed in baseline/_ref."""
    import multiprocessing as mp
    import sys

    ref_site = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_site, "shockhash")):
        pytest.skip("reference package not installed in baseline/_ref")
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refbuild

    if not refbuild.have_ref():
        pytest.skip("oracle/_ref not built")
    if ref_site not in sys.path:
        sys.path.insert(0, ref_site)
    import shockhash

    from paper_2308_09561_b200 import workloads as W

    keys = W.keys_as_bytes(W.raw_keys(4, 100_000))
    stock = shockhash.build(keys, 2000, 40).serialize()
    with mp.get_context("fork").Pool(min(8, os.cpu_count() or 1)) as pool:
        mine = refbuild.build_descriptor_ref(keys, 2000, 40, pool)
    assert mine == stock
