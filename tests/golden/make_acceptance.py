"""Golden values for tests/test_gpu_acceptance.py from the REAL reference
(compiled backend; see make_golden.py for the out-of-tree build):

    PYTHONPATH=/tmp/refpkg python tests/golden/make_acceptance.py

The reference's acceptance suite builds on synthetic_keys(10**6, 42)
(pkg/tests/test_acceptance.py); here the same inputs are run through the
reference's build/query and trial statistics and the outputs are pinned
(descriptor sha256, bits/key, query sha, mean seeds), so the GPU tests can
require identical results, not only the acceptance thresholds."""

import hashlib
import json
import os
import sys
import time

import numpy as np

import shockhash_ref as ref
from shockhash_ref import experiments as ex
from shockhash_ref.keys import synthetic_hashed, synthetic_keys

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(b):
    return hashlib.sha256(b).hexdigest()


def main():
    assert ref.BACKEND_NAME == "compiled"
    out = {"builds": [], "trials": [], "retrieval": None}
    keys = synthetic_keys(10**6, 42)
    for N, n, b in ((10**3, 16, 100), (10**3, 24, 2000), (10**5, 24, 2000), (10**6, 30, 2000), (10**6, 24, 2000),
                    (10**6, 36, 2000)):
        t = time.time()
        d = ref.build(keys[:N], b, n, ref.MODE_ROTATE)
        blob = d.serialize()
        q = d.query_many(keys[:N])
        out["builds"].append(dict(N=N, n=n, b=b, desc_sha=sha(blob), bits_per_key=d.stats()["bits_per_key"],
                                  query_sha=sha(np.asarray(q, "<u8").tobytes()), seconds=time.time() - t))
        print(out["builds"][-1], file=sys.stderr, flush=True)
    for ns, mode in (([8], "bruteforce"), ([10, 16, 20], "plain"), ([16, 24, 30], "rotate")):
        for r in ex.trial_statistics(ns, mode, 10**4, seed=1):
            out["trials"].append(dict(n=r.n, mode=r.mode, reps=r.reps, mean_seed=r.mean_seed,
                                      mean_log2_seed=r.mean_log2_seed, overhead_bits=r.overhead_bits))
            print(out["trials"][-1], file=sys.stderr, flush=True)
    N = 10**7
    hi, lo = synthetic_hashed(N, 2024)
    from shockhash_ref._kernels import get_backend

    K = get_backend("compiled")
    rhs = (K.mix64_batch(hi) & np.uint64(1)).astype(np.uint8)
    from shockhash_ref import retrieval

    t = time.time()
    sys_ = retrieval.retrieval_build_arrays(hi, lo, rhs)
    out["retrieval"] = dict(N=N, gen=2024, seed=int(sys_.seed), m=int(sys_.m), size_bits=int(sys_.size_bits),
                            words_sha=sha(np.asarray(sys_.words, "<u8").tobytes()), seconds=time.time() - t)
    print(out["retrieval"], file=sys.stderr, flush=True)
    with open(os.path.join(HERE, "acceptance.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
