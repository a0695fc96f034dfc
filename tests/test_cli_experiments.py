"""The CLI (cli.py) and the experiments module (experiments.py) against the
reference's outputs (tests/golden/experiments.json, made by running the real
reference) and its own CLI/experiment tests (tests/test_cli.py,
tests/test_experiments.py of the reference)."""

import math
from fractions import Fraction

import pytest

from conftest import golden
from paper_2308_09561_b200 import cli
from paper_2308_09561_b200 import experiments as ex
from paper_2308_09561_b200.errors import InvalidParameterError

gpu = pytest.mark.gpu


# ---------------------------------------------------------------- host only


def test_parse_n_range():
    assert cli._parse_n_range("16") == [16]
    assert cli._parse_n_range("6..12") == [6, 8, 10, 12]
    assert cli._parse_n_range("1..3..1") == [1, 2, 3]
    with pytest.raises(InvalidParameterError):
        cli._parse_n_range("9..5")


def test_usage_error_exit_code(capsys):
    with pytest.raises(SystemExit) as ei:
        cli.main(["build", "--synthetic", "10"])  # missing --out
    assert ei.value.code == cli.EXIT_USAGE
    capsys.readouterr()


def test_bad_range_exit_code(capsys):
    assert cli.main(["experiment", "trials", "--n", "9..5", "--reps", "10"]) == cli.EXIT_USAGE
    capsys.readouterr()


def test_analytic_helpers():
    assert ex.bijection_probability(1) == pytest.approx(1.0)
    assert ex.bijection_probability(3) == pytest.approx(6 / 27)
    assert ex.lower_bound_bits(3) == pytest.approx(-math.log2(6 / 27))
    assert ex.d_recurrence(1) == pytest.approx(2.0)
    assert ex.d_recurrence(2) == pytest.approx(8 / 3)
    for n in (1, 2, 4, 16, 64, 256, 1024):
        assert ex.d_recurrence(n) <= math.e * math.sqrt(2 * n) + 1e-9
    vals = [ex.filter_pass_bound(n) for n in range(2, 65)]
    assert all(b < a for a, b in zip(vals, vals[1:]))
    assert ex.filter_pass_bound(64) < 2**-13


def test_mc_component_factor_golden():
    for r in golden("experiments.json")["component"]:
        assert ex.mc_component_factor(r["n"], r["trials"], r["seed"]) == r["value"]


def test_parameter_validation():
    with pytest.raises(InvalidParameterError):
        ex.trial_statistics([4], "nope", 10)
    with pytest.raises(InvalidParameterError):
        ex.trial_statistics([4], "plain", 0)
    with pytest.raises(InvalidParameterError):
        ex.trial_statistics([20], "bruteforce", 10)
    with pytest.raises(InvalidParameterError):
        ex.exact_pseudoforest_probability(0)
    with pytest.raises(InvalidParameterError):
        ex.exact_pseudoforest_probability(ex.ENUM_MAX_N + 1)
    with pytest.raises(InvalidParameterError):
        ex.mc_filter_pass(65, 10)


# ---------------------------------------------------------------- GPU


@gpu
def test_trial_statistics_golden():
    """One batched launch per n gives the reference's per-leaf statistics."""
    by_cfg = {}
    for r in golden("experiments.json")["trial_statistics"]:
        by_cfg.setdefault((r["mode"], r["reps"], r["seed"]), []).append(r)
    for (mode, reps, seed), recs in by_cfg.items():
        rows = ex.trial_statistics([r["n"] for r in recs], mode, reps, seed)
        for row, r in zip(rows, recs):
            assert (row.n, row.mode, row.reps) == (r["n"], r["mode"], r["reps"])
            assert row.mean_seed == r["mean_seed"], r
            assert row.mean_log2_seed == r["mean_log2_seed"], r
            assert row.overhead_bits == pytest.approx(r["overhead_bits"], rel=1e-12, abs=1e-12), r


@gpu
def test_filter_and_enumeration_golden():
    g = golden("experiments.json")
    for r in g["filter_pass"]:
        assert ex.mc_filter_pass(r["n"], r["trials"], r["seed"]) == r["value"]
    for r in g["enumerate"]:
        n = r["n"]
        assert ex.exact_pseudoforest_probability(n) == Fraction(r["pf_count"], n ** (2 * n))
        assert ex.exact_mean_orientations(n) == Fraction(r["sum_2c"], n ** (2 * n))
    assert ex.exact_pseudoforest_probability(2) == Fraction(7, 8)
    for n in range(1, ex.ENUM_MAX_N + 1):
        assert ex.exact_mean_orientations(n) == ex.exact_mean_orientations_closed_form(n)
        p = float(ex.exact_pseudoforest_probability(n))
        assert p >= max(ex.pf_probability_lower_bounds(n))
    slope, _ = ex.filter_slope([8, 12, 16, 20], 20000, 1)
    assert slope < 0
    with pytest.raises(InvalidParameterError):
        ex.filter_slope([64], 10)


@gpu
def test_cli_build_verify_synthetic(tmp_path, capsys):
    out = tmp_path / "d.mph"
    assert cli.main(["build", "--synthetic", "2000", "--b", "200", "--n", "16", "--out", str(out)]) == cli.EXIT_OK
    text = capsys.readouterr().out
    assert "keys: 2000" in text and "bits/key" in text and "backend=cuda" in text
    assert cli.main(["verify", str(out), "--synthetic", "2000"]) == cli.EXIT_OK
    assert "verified: 2000" in capsys.readouterr().out


@gpu
def test_cli_build_verify_file_and_failures(tmp_path, capsys):
    from paper_2308_09561_b200.keys import synthetic_keys

    keyfile = tmp_path / "keys.txt"
    keyfile.write_bytes(b"\n".join(synthetic_keys(500, 3)) + b"\n")
    out = tmp_path / "d.mph"
    assert cli.main(["build", "--input", str(keyfile), "--b", "100", "--n", "12", "--out", str(out)]) == cli.EXIT_OK
    assert cli.main(["verify", str(out), "--input", str(keyfile)]) == cli.EXIT_OK
    # other keys, same count / different count
    assert cli.main(["verify", str(out), "--synthetic", "500", "--gen-seed", "1"]) == cli.EXIT_VERIFY
    assert cli.main(["verify", str(out), "--synthetic", "400"]) == cli.EXIT_VERIFY
    # corrupted descriptor
    out2 = tmp_path / "e.mph"
    cli.main(["build", "--synthetic", "1000", "--out", str(out2), "--n", "16", "--b", "100"])
    blob = bytearray(out2.read_bytes())
    blob[len(blob) // 2] ^= 0x10
    out2.write_bytes(bytes(blob))
    assert cli.main(["verify", str(out2), "--synthetic", "1000"]) == cli.EXIT_VERIFY
    # duplicates, missing input, bad leaf size
    dup = tmp_path / "dup.txt"
    dup.write_bytes(b"aaa\nbbb\naaa\n")
    assert cli.main(["build", "--input", str(dup), "--b", "100", "--n", "8", "--out", str(tmp_path / "x")]) == \
        cli.EXIT_DUPLICATE
    assert "duplicate" in capsys.readouterr().err
    assert cli.main(["build", "--input", str(tmp_path / "missing.txt"), "--out", str(tmp_path / "y")]) == cli.EXIT_IO
    assert cli.main(["build", "--synthetic", "100", "--n", "80", "--b", "100", "--out", str(tmp_path / "z")]) == \
        cli.EXIT_USAGE
    capsys.readouterr()


@gpu
def test_verify_reports_first_offender():
    """verify's offender is the first key (input order) whose index repeats an
    earlier key's, as the reference's sequential scan reports it."""
    from paper_2308_09561_b200 import recsplit
    from paper_2308_09561_b200.keys import synthetic_keys

    keys = synthetic_keys(3000, 11)
    desc = recsplit.build(keys, 300, 16)
    assert desc.verify(keys) == (True, None)
    other = synthetic_keys(3000, 12)
    ok, off = desc.verify(other)
    out = [int(x) for x in desc.query_many(other)]
    seen, expect = set(), None
    for i, v in enumerate(out):
        if v >= len(keys) or v in seen:
            expect = other[i]
            break
        seen.add(v)
    assert not ok and off == expect


@gpu
def test_cli_experiments(tmp_path, capsys):
    csvf = tmp_path / "t.csv"
    assert cli.main(["experiment", "trials", "--n", "4..6", "--reps", "50", "--csv", str(csvf)]) == cli.EXIT_OK
    assert capsys.readouterr().out.splitlines()[0].startswith("n,mode,reps")
    assert len(csvf.read_text().strip().splitlines()) == 3
    assert cli.main(["experiment", "enumerate", "--n", "1..3..1"]) == cli.EXIT_OK
    out = capsys.readouterr().out.splitlines()
    assert out[0].startswith("n,pf_probability") and len(out) == 4
    assert cli.main(["experiment", "filter", "--n", "8", "--trials", "2000"]) == cli.EXIT_OK
    assert cli.main(["experiment", "component", "--n", "8", "--trials", "2000"]) == cli.EXIT_OK
    assert cli.main(["bench", "--n", "10", "--reps", "5"]) == cli.EXIT_OK
    assert "backend,op,n,reps" in capsys.readouterr().out
