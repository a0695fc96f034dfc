"""bench.py's multi-GPU launcher: ``--gpus N`` with no WORLD_SIZE re-launches
itself under torch.distributed.run with N ranks and prints ONE JSON line
with ``n_gpus: N``.  On this one-GPU box the ranks share the GPU over gloo
(``SHK_DIST_BACKEND=gloo``); the line must still carry the reference's C4
descriptor sha (every rank's replicated descriptor) and the sha of the 1e8
query outputs answered by the three ranks' batch ranges."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu


def test_bench_gpus3_launches_three_ranks():
    env = dict(os.environ, SHK_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, "bench.py", "--gpus", "3", "--steps", "1", "--warmup", "1", "--leaf-configs", "1,3",
           "--no-c2", "--no-cpu-baseline", "--query-reps", "1"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 3
    assert d["parity"]["desc_sha256"] == golden("c4.json")["desc_sha"]
    assert d["parity"]["desc_matches_reference"] and d["parity"]["e2e_desc_matches_reference"]
    assert d["query"]["ranks"] == 3 and d["query"]["matches_reference"]
    for c in ("C1", "C3"):
        p = d["leaf_search"][c]["parity"]
        assert p["seed_mismatches"] == 0 and p["fbits_mismatches"] == 0 and p["leaves_checked"] == p["of_leaves"]
