#!/usr/bin/env python3
"""Benchmark: ShockHash-RS MPHF build on B200 (BASELINE.json configs[3], "C4").

Workload (one step): build the minimal perfect hash function of N=10,000,000
uniform random 64-bit keys (8-byte little-endian strings, ``default_rng(4)``),
leaf size n=40, bucket size b=2000, rotation fitting — the largest
single-GPU configuration of BASELINE.json.  Reported beside it: the 1e8
queries of the same config, the leaf-only configs C1/C3/C5, the C2 build and
its 1e6 queries, the measured integer-issue peak, and the reference's CPU
path timed on this host.

  value : keys/s of the build from master hash codes resident in HBM
          (bucketize -> split searches -> leaf searches + orientation ->
          Rice stream -> ribbon), CUDA events on the launching stream.
  e2e   : keys/s through the public C-ABI/Python API with HOST buffers:
          8-byte key blob H2D -> blake2b -> build -> descriptor bytes D2H.

Multi-GPU: ``--gpus N`` with no WORLD_SIZE in the environment re-launches
itself under ``torch.distributed.run`` with N ranks (one per GPU, NCCL).
Buckets are sharded by range over ranks (strong scaling, total N fixed); one
all-gather joins streams and choice bits; the ranks solve the global ribbon
column-sharded (dist.ribbon_sharded) and every rank ends with the whole
descriptor.  Queries: replicated descriptor, batch sharded by range.  Leaf
configs C3/C5: one leaf queue shared by all ranks (a CUDA IPC counter, see
dist.SharedLeafQueue); C1: contiguous leaf ranges.  Time = max over ranks.
``SHK_DIST_BACKEND=gloo`` runs the N ranks on one GPU (functional check).

``--impl reference`` times the reference's CPU implementation of the same
path: its own compiled kernels (oracle/_ref, built from /root/reference by
oracle/build_ref.sh) under the reference's build orchestration restated in
oracle/refbuild.py, with all host cores over buckets, on a bounded sample.
"""

import argparse
import gc
import hashlib
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(N=10_000_000, n=40, b=2000, mode=1, queries=100_000_000)
CFG2 = dict(N=100_000, n=24, b=500, mode=1, queries=1_000_000)
W_KEY = 53   # int32 ops per key-hash-eval, 64-bit masks
W_SEED = 22  # per seed mixer + mask compare
W_ROT = 10   # per rotation test, 64-bit masks
W_SPLIT = 46  # per split key-eval
W_QUERY = 620  # int32 ops per query with the derived node index
INT_OPS_PER_CLK_SM = 128  # 4 SMSPs x 32 lanes, ALU + FMA pipes (one warp-instr/clk/SMSP)
MAX_MHZ = 1965.0
HBM_FALLBACK_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
C3_FIG2_MEAN = 4023  # PAPER.md:788, plain ShockHash n=32
C3_RICE_MODEL = 4984  # (e/2)^n * e / sqrt(pi n) at n=32 (recsplit.py:173-184)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.rows = []
        self.gpu = gpu_index
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *e):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        sm = []
        mx = None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() in ("active", "1", "yes"):
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_info():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


DIST_BACKEND = os.environ.get("SHK_DIST_BACKEND", "nccl")  # gloo: functional runs of N ranks sharing one GPU


def coll_device():
    import torch

    return torch.device("cuda", torch.cuda.current_device()) if DIST_BACKEND == "nccl" else torch.device("cpu")


def reduce_over_ranks(x, world, op="max"):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(x)], dtype=torch.float64, device=coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def max_over_ranks(x, world):
    return reduce_over_ranks(x, world, "max")


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def sha_rank_order(arr, world):
    """sha256 of the concatenation of every rank's array in rank order
    (rank 0 returns it; the slices travel to rank 0 one at a time)."""
    h = hashlib.sha256()
    raw = np.ascontiguousarray(arr).view(np.uint8)
    if world == 1:
        h.update(raw.tobytes())
        return h.hexdigest()
    import torch
    import torch.distributed as dist

    dev = coll_device()
    rank = dist.get_rank()
    n = torch.tensor([raw.size], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, n)
    if rank == 0:
        h.update(raw.tobytes())
        for r in range(1, world):
            buf = torch.empty(max(int(sizes[r].item()), 1), dtype=torch.uint8, device=dev)
            dist.recv(buf, src=r)
            h.update(buf[: int(sizes[r].item())].cpu().numpy().tobytes())
        return h.hexdigest()
    t = torch.from_numpy(raw.copy() if raw.size else np.zeros(1, np.uint8)).to(dev)
    dist.send(t, dst=0)
    return None


def gather_ints(x, world):
    """[x of rank 0, x of rank 1, ...] on every rank."""
    if world == 1:
        return [x]
    import torch
    import torch.distributed as dist

    t = torch.tensor([int(x)], dtype=torch.int64, device=coll_device())
    out = [torch.zeros(1, dtype=torch.int64, device=coll_device()) for _ in range(world)]
    dist.all_gather(out, t)
    return [int(o.item()) for o in out]


def input_keys():
    from paper_2308_09561_b200 import workloads as W

    k = W.build_keys(4)
    blob = np.frombuffer(np.ascontiguousarray(k, dtype="<u8").tobytes(), dtype=np.uint8)
    return k, blob


def hbm_peak():
    """(GB/s, source) — the driver-measured copy bandwidth, else the fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


NCU_TREE_SUMMARY = os.path.join(ROOT, "profiles", "ncu_tree_latest.csv")


def ncu_traffic():
    """DRAM bytes (read + write) per launch of the tree kernel from the
    committed `ncu --set full` summary (tools/summarize_ncu.py), or None."""
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    try:
        import csv

        tot = 0.0
        seen = 0
        with open(NCU_TREE_SUMMARY) as f:
            for r in csv.DictReader(f):
                if r["kernel"].startswith("void tree_kernel") and r["metric"] in ("dram__bytes_read.sum",
                                                                                  "dram__bytes_write.sum"):
                    tot += float(r["value"]) * scale.get(r.get("unit", "byte"), 1)
                    seen += 1
        return int(tot) if seen == 2 else None
    except (OSError, KeyError, ValueError):
        return None


def measure_int_peak(dev, sms):
    """The integer-issue microbenchmark (csrc/shk_peak.cu) next to the nominal
    128 ops/clk/SM: Tops/s per instruction mix, best = the measured peak."""
    res = {}
    for kind, name in dev.INT_PEAK_KINDS.items():
        ms, ops = dev.int_peak(kind, 16384)
        res[name] = round(ops / (ms * 1e-3) / 1e12, 3)
    nominal = INT_OPS_PER_CLK_SM * sms * MAX_MHZ * 1e6 / 1e12
    best = max(res.values())
    return {"nominal_Tops": round(nominal, 2), "measured_Tops": res, "measured_best_Tops": best,
            "measured_over_nominal": round(best / nominal, 4),
            "how": "8 independent 32-bit chains per thread, 64 warps/SM, one timed launch per mix "
                   "(inline PTX: lop3.b32 -> LOP3, mad.lo.u32 -> IMAD, shf.r.wrap -> SHF)"}


def roofline_numbers(prof, hash_evals, n, clock_mhz, sms, int_peak=None):
    """Integer-issue roofline of the dominant kernel (split or leaf search)."""
    ph = prof["phase_ms"]
    leaf_ops = hash_evals * W_KEY + (hash_evals / 2) * W_ROT + (hash_evals / (2 * n)) * 2 * W_SEED
    split_ops = prof["split_evals"] * W_SPLIT
    peak = INT_OPS_PER_CLK_SM * sms * MAX_MHZ * 1e6 / 1e12  # Tops/s at max clock
    if ph["leaf_search"] < 0.05 * ph["split_search"]:
        # persistent schedule: split and leaf searches share one kernel launch
        # (and its tail: tree_resume_kernel, the leaves handed off when the
        # queue ran dry -- both inside the timed phase)
        kern = {"tree_kernel+tree_resume_kernel(split+leaf search)": (leaf_ops + split_ops,
                                                                      ph["split_search"] + ph["leaf_search"])}
    else:
        kern = {
            "leaf_search": (leaf_ops, ph["leaf_search"]),
            "split_search": (split_ops, ph["split_search"]),
        }
    dom = max(kern, key=lambda k: kern[k][1])
    ops, ms = kern[dom]
    ach = ops / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
    other = {k: {"achieved": round(v[0] / (v[1] * 1e-3) / 1e12, 3) if v[1] > 0 else None,
                 "ms": round(v[1], 3), "algorithmic_ops": int(v[0])} for k, v in kern.items()}
    out = {
        "kernel": dom,
        "bound": "int32-issue",
        "achieved": round(ach, 3),
        "peak": round(peak, 2),
        "unit": "Tops/s",
        "frac": round(ach / peak, 4),
        "traffic": ncu_traffic() if dom.startswith("tree_kernel") else None,
        "traffic_unit": "bytes per launch (dram read + write, profiles/ncu_tree_latest.csv)",
        "peak_source": "nominal 128 int32 ops/clk/SM x %d SMs x 1965 MHz (MEASURED_PEAKS.json has no integer "
                       "peak; the measured microbenchmark peak is int_peak_measured)" % sms,
        "frac_at_run_clock": round(ach / (peak * clock_mhz / MAX_MHZ), 4) if clock_mhz else None,
        "per_kernel": other,
    }
    if int_peak:
        out["int_peak_measured"] = int_peak["measured_best_Tops"] * sms / int_peak["sms"]
        out["frac_of_measured"] = round(ach / out["int_peak_measured"], 4)
    return out


def cpu_baseline_sample(seconds_target=15.0):
    """Reference CPU path on a bounded sample of the same workload (rank 0)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refbuild

    return refbuild.time_build_sample(seconds_target=seconds_target)


def init_dist(world, local):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local if DIST_BACKEND == "nccl" else 0)
    if DIST_BACKEND == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        os.environ["SHK_DEVICE"] = "0"
        dist.init_process_group(DIST_BACKEND)


def run_ours(args):
    rank, world, local = dist_info()
    os.environ.setdefault("SHK_DEVICE", str(local))
    # SHK_FORCE_SHARDED=1 runs the sharded (NCCL) path even at world size 1
    sharded = world > 1 or os.environ.get("SHK_FORCE_SHARDED") == "1"
    if sharded:
        init_dist(world, local)
    from paper_2308_09561_b200 import dist as shdist
    from paper_2308_09561_b200 import device as dev
    from paper_2308_09561_b200 import recsplit

    N, n, b = CFG["N"], CFG["n"], CFG["b"]
    k, blob = input_keys()
    sms = dev.num_sms()
    int_peak = measure_int_peak(dev, sms)
    int_peak["sms"] = sms
    # N > 1: each rank holds only its slice of the keys (input-sharded build,
    # two all-to-alls); SHK_SHARD_INPUT=0: every rank holds all keys
    # (replicated fingerprinting and bucket sort)
    input_sharded = sharded and os.environ.get("SHK_SHARD_INPUT", "1") != "0"
    k0, k1 = ((N * rank) // world, (N * (rank + 1)) // world) if input_sharded else (0, N)
    n_loc = k1 - k0
    my_blob = blob[8 * k0 : 8 * k1]
    # resident inputs: the master codes (of this rank's keys), computed once on the GPU
    d_blob = dev.DeviceBuffer.from_host(my_blob)
    d_hi = dev.DeviceBuffer(8 * n_loc)
    d_lo = dev.DeviceBuffer(8 * n_loc)
    dev.blake2b_fixed_device(d_blob, 8, n_loc, 0, d_hi, d_lo)
    d_blob.free()
    dev.sync()

    def step():
        if not sharded:
            d = recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, b, n, CFG["mode"])
            return d, d.device_profile
        if input_sharded:
            d, prof = shdist.build_hashed_device_sharded_input(d_hi.ptr, d_lo.ptr, n_loc, N, b, n, CFG["mode"],
                                                               device=coll_device())
        else:
            d, prof = shdist.build_hashed_device_sharded(d_hi.ptr, d_lo.ptr, N, b, n, CFG["mode"],
                                                         device=coll_device())
        prof = dict(prof)
        prof["phase_ms"] = dict(zip(("bucketize", "split_search", "leaf_search", "rice", "ribbon"), prof["phase_ms"]))
        return d, prof

    # One untimed instrumented build counts the reference's split `evals`
    # (algorithmic work of the split searches; the timed builds run the
    # verdict-only search, identical seeds).
    dev.set_option(dev.OPT_EXACT_SPLIT_EVALS, 1)
    _, prof_exact = step()
    dev.set_option(dev.OPT_EXACT_SPLIT_EVALS, 0)
    split_evals_exact = prof_exact["split_evals"]
    for _ in range(args.warmup):
        desc, prof = step()
    parity = {}
    gpath = os.path.join(ROOT, "tests", "golden", "c4.json")
    g4 = json.load(open(gpath)) if os.path.exists(gpath) else None
    blob_desc = desc.serialize()
    parity["desc_sha256"] = hashlib.sha256(blob_desc).hexdigest()
    if g4:
        ok = parity["desc_sha256"] == g4["desc_sha"]
        parity["desc_matches_reference"] = bool(reduce_over_ranks(1.0 if ok else 0.0, world, "sum") == world)
        if world > 1:
            parity["desc_matches_reference_on_ranks"] = world if parity["desc_matches_reference"] else "some ranks differ"
    parity["bits_per_key"] = round(len(blob_desc) * 8 / N, 6)
    barrier(world)
    dev.sync()
    launches0 = dev.launch_count()
    with ClockSampler(local) as clk:
        barrier(world)
        dev.sync()
        t_wall = time.perf_counter()
        with dev.timer() as tm:
            profs = []
            for _ in range(args.steps):
                desc, prof = step()
                profs.append(prof)
        dev.sync()
        wall = time.perf_counter() - t_wall
        barrier(world)
    launches = dev.launch_count() - launches0
    ms_total = max_over_ranks(tm.ms, world)
    ms_step = ms_total / args.steps
    value = N / (ms_step * 1e-3)

    # e2e through the public API with host buffers: the caller's pinned key
    # blob in, serialized descriptor bytes out; max wall over ranks
    desc_bytes = 0
    out = None
    pinned = dev.PinnedBuffer.from_array(my_blob)  # the caller's key buffer (this rank's slice), page-locked

    def e2e_step():
        if input_sharded:
            d2, _ = shdist.build_blob_sharded_input(pinned.array, 8, N, b, n, CFG["mode"], device=coll_device())
        elif sharded:
            d2, _ = shdist.build_blob_sharded(pinned.array, 8, b, n, CFG["mode"], device=coll_device())
        else:
            d2 = recsplit.build_blob(pinned.array, 8, b, n, CFG["mode"])
        return d2.serialize()

    e2e_step()  # warm-up of the host-buffer path (copy stream, events, pinned pages)
    dev.sync()
    barrier(world)
    gc.collect()
    gc.disable()  # no collector pauses inside the timed host-side region
    try:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            out = e2e_step()
            desc_bytes = len(out)
        e2e_s = (time.perf_counter() - t0) / args.steps
    finally:
        gc.enable()
    e2e_s = max_over_ranks(e2e_s, world)
    e2e = {"value": round(N / e2e_s, 1), "unit": "keys/s", "h2d_bytes_per_step": int(my_blob.nbytes) * world,
           "d2h_bytes_per_step": int(desc_bytes), "ms_per_step": round(e2e_s * 1e3, 3),
           "path": ("dist.build_blob_sharded_input" if input_sharded else
                    "dist.build_blob_sharded" if sharded else "recsplit.build_blob")
           + "(pinned host 8-byte key blob) -> serialize(); H2D+blake2b+build+D2H timed"
           + (", max wall over ranks" if world > 1 else "")}
    pinned.free()
    if args.check and out is not None:
        parity["e2e_desc_matches_reference"] = hashlib.sha256(out).hexdigest() == parity.get("desc_sha256")

    # algorithmic work of the timed step summed over ranks (roofline)
    hash_evals_local = prof.get("hash_evals")
    if hash_evals_local is None and desc is not None and desc.build_stats:
        hash_evals_local = desc.build_stats.get("hash_evals")
    hash_evals_all = reduce_over_ranks(hash_evals_local or 0, world, "sum")
    split_evals_all = reduce_over_ranks(split_evals_exact, world, "sum")
    tree_ms_max = max_over_ranks(prof["phase_ms"]["split_search"] + prof["phase_ms"]["leaf_search"], world)
    bucket_ms = max_over_ranks(prof["phase_ms"]["bucketize"], world)

    # queries (C4: 1e8 keys drawn from the set): replicated descriptor, batch
    # sharded by range over the ranks, device-resident
    query = None
    if args.queries > 0:
        query = bench_queries(desc, k, args, dev, sms, rank, world, int_peak)
    leaf_lines = {}
    if args.leaf_configs:
        for cfg in [int(x) for x in args.leaf_configs.split(",") if x]:
            leaf_lines[f"C{cfg}"] = bench_leaf(cfg, args, dev, sms, rank, world, int_peak)
    c2 = bench_c2(args, dev, rank) if (args.c2 and rank == 0) else None

    if rank != 0:
        return
    prof = dict(profs[-1])
    # roofline inputs: work summed over ranks, the dominant kernel's time the
    # max over ranks (at N = 1 these are the rank's own numbers)
    prof["split_evals"] = split_evals_all
    prof["phase_ms"] = dict(prof["phase_ms"])
    if world > 1:
        prof["phase_ms"]["split_search"], prof["phase_ms"]["leaf_search"] = tree_ms_max, 0.0
    hash_evals = hash_evals_all if hash_evals_all else None
    clocks = clk.summary()
    hbm, hbm_src = hbm_peak()
    line = {
        "metric": "keys/s MPHF build (ShockHash-RS, N=1e7, n=40, b=2000, rotate)",
        "value": round(value, 1),
        "unit": "keys/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic: default_rng(4) uniform 64-bit keys as 8-byte LE strings (the reference's recipe, SURVEY.md §8(d))",
        "config": {"workload": "C4: ShockHash-RS build N=10,000,000, leaf n=40, bucket b=2000, mode rotate, eps=0.05",
                   "N": N, "n": n, "b": b,
                   "parallelism": ((f"bucket-range x{world} ({DIST_BACKEND}), "
                                    + ("input-sharded: keys -> bucket owners, rows -> column owners (all-to-all)"
                                       if input_sharded else "replicated input"))
                                   if world > 1 else "single GPU"),
                   "l2": "inputs 160 MB of resident master codes + 160 MB working keys > 126 MB L2 (no flush needed)"},
        "clocks": clocks,
        "gpu_launches": int(launches),
        "wall_s_timed": round(wall, 3),
        "phase_ms": {k2: round(v, 3) for k2, v in prof["phase_ms"].items()},
        "parity": parity,
        "e2e": e2e,
    }
    if hash_evals is not None:
        line["roofline"] = roofline_numbers(prof, hash_evals, n, clocks.get("sm_mhz"), sms * world, int_peak)
        if world > 1:
            line["roofline"]["peak_source"] += f" (all {world} GPUs)"
    line["int_peak"] = {k2: v for k2, v in int_peak.items() if k2 != "sms"}
    # bucketing (a3): 32 algorithmic bytes per key (read hi/lo, write sorted hi/lo)
    nb_keys = N if (world == 1 or not input_sharded) else (N + world - 1) // world  # keys one rank sorts
    line["bucketize"] = {"ms": round(bucket_ms, 3), "algorithmic_bytes": 32 * nb_keys,
                         "GBps": round(32 * nb_keys / (bucket_ms * 1e-3) / 1e9, 1),
                         "hbm_frac": round(32 * nb_keys / (bucket_ms * 1e-3) / 1e9 / hbm, 4), "hbm_peak_GBps": hbm,
                         "peak_source": hbm_src,
                         "note": ("each rank sorts the keys of its bucket range (max over ranks)" if input_sharded
                                  else "every rank bucket-sorts all N keys" if world > 1 else "single GPU")}
    if query:
        line["query"] = query
    if leaf_lines:
        line["leaf_search"] = leaf_lines
    if c2:
        line["c2"] = c2
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline_sample(args.cpu_seconds)
        except Exception as e:  # report, never crash the GPU line
            line["cpu_baseline"] = {"error": f"{type(e).__name__}: {e}"}
        if not args.no_cpu_leaf:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import refleaf

            for cfg in [int(x) for x in args.leaf_configs.split(",") if x]:
                try:
                    leaf_lines[f"C{cfg}"]["cpu_baseline"] = refleaf.time_leaf_config(cfg)
                except Exception as e:
                    leaf_lines[f"C{cfg}"]["cpu_baseline"] = {"error": f"{type(e).__name__}: {e}"}
            if c2:
                try:
                    import refbuild

                    c2["cpu_baseline"] = refbuild.time_build_c2()
                except Exception as e:
                    c2["cpu_baseline"] = {"error": f"{type(e).__name__}: {e}"}
    print(json.dumps(line), flush=True)


def bench_queries(desc, k, args, dev, sms, rank, world, int_peak):
    """1e8 C4 queries: every rank holds the whole descriptor and answers the
    range [Q r/W, Q (r+1)/W) of the batch (no exchange); time = max over
    ranks.  Outputs are hashed in rank order on rank 0 for parity."""
    from paper_2308_09561_b200 import workloads as W

    Q = args.queries
    q0, q1 = (Q * rank) // world, (Q * (rank + 1)) // world
    Qr = q1 - q0
    idx = W.query_indices(4, Q)[q0:q1]
    # master codes of the query keys (blake2b on the GPU from the key bytes)
    qblob = np.frombuffer(np.ascontiguousarray(k[idx], dtype="<u8").tobytes(), dtype=np.uint8)
    d_qblob = dev.DeviceBuffer.from_host(qblob)
    d_qhi = dev.DeviceBuffer(8 * max(Qr, 1))
    d_qlo = dev.DeviceBuffer(8 * max(Qr, 1))
    dev.blake2b_fixed_device(d_qblob, 8, Qr, desc.salt, d_qhi, d_qlo)
    d_qblob.free()
    d_out = dev.DeviceBuffer(8 * max(Qr, 1))
    dd = desc.device()
    dd.query_device(d_qhi.ptr, d_qlo.ptr, Qr, d_out.ptr)  # warm-up; node index decoded once per descriptor
    dev.sync()
    barrier(world)
    reps = max(1, args.query_reps)
    with dev.timer() as tm:
        for _ in range(reps):
            dd.query_device(d_qhi.ptr, d_qlo.ptr, Qr, d_out.ptr)
    ms = max_over_ranks(tm.ms / reps, world)
    res = {"queries": Q, "value": round(Q / (ms * 1e-3), 1), "unit": "queries/s", "ms": round(ms, 3),
           "ranks": world, "sharding": "replicated descriptor, batch range per rank" if world > 1 else "single GPU"}
    hbm, hbm_src = hbm_peak()
    gbs = 24.0 * Q / (ms * 1e-3) / 1e9
    res["hbm_GBps_algorithmic"] = round(gbs, 1)
    res["hbm_frac"] = round(gbs / (hbm * world), 4)
    res["hbm_peak_source"] = hbm_src
    nominal = INT_OPS_PER_CLK_SM * sms * world * MAX_MHZ * 1e6 / 1e12
    ach = W_QUERY * Q / (ms * 1e-3) / 1e12
    res["int_roofline"] = {"achieved": round(ach, 3), "peak": round(nominal, 2), "unit": "Tops/s",
                           "frac": round(ach / nominal, 4),
                           "frac_of_measured": round(ach / (int_peak["measured_best_Tops"] * world), 4),
                           "work": f"{W_QUERY} int32 ops per query (SURVEY.md §8(d), derived node index)"}
    res["untimed"] = "node_index_kernel (Rice stream decoded once per descriptor, ~70 us at C4) runs in the warm-up"
    # e2e through the public API with host buffers: the query keys' 8-byte
    # strings (pinned) in, indices out (MphfDescriptor.query_blob: H2D,
    # blake2b, query, D2H pipelined in chunks); max wall over ranks
    pinned = dev.PinnedBuffer.from_array(qblob)
    hout = dev.PinnedBuffer(8 * max(Qr, 1), dtype=np.uint64)
    desc.query_blob(pinned.array, 8, out=hout.array[:Qr])  # warm-up
    barrier(world)
    t0 = time.perf_counter()
    desc.query_blob(pinned.array, 8, out=hout.array[:Qr])
    e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    res["e2e"] = {"value": round(Q / e2e_s, 1), "unit": "queries/s", "ms": round(e2e_s * 1e3, 3),
                  "h2d_bytes": 8 * Q, "d2h_bytes": 8 * Q,
                  "path": "MphfDescriptor.query_blob(pinned 8-byte keys) -> indices in pinned host memory"}
    e2e_ok = None
    if args.check:
        out = d_out.download(np.uint64, Qr)
        e2e_ok = bool((hout.array[:Qr] == out).all())
        qsha = sha_rank_order(out.astype("<u8"), world)
        gpath = os.path.join(ROOT, "tests", "golden", "c4.json")
        if rank == 0 and os.path.exists(gpath) and Q == CFG["queries"]:
            res["matches_reference"] = qsha == json.load(open(gpath))["query_sha"]
        res["e2e"]["outputs_equal_device_path"] = bool(reduce_over_ranks(1.0 if e2e_ok else 0.0, world, "sum") == world)
    pinned.free()
    hout.free()
    for b_ in (d_qhi, d_qlo, d_out):
        b_.free()
    return res


def leaf_golden(cfg):
    """Full-population reference goldens (tests/golden/c{cfg}_full.bin, every
    leaf: seed, f bits), else the small json sample."""
    full = os.path.join(ROOT, "tests", "golden", f"c{cfg}_full.bin")
    if os.path.exists(full):
        meta = json.load(open(os.path.join(ROOT, "tests", "golden", f"c{cfg}_full.json")))
        raw = open(full, "rb").read()
        if hashlib.sha256(raw).hexdigest() != meta["file_sha256"]:
            raise RuntimeError(f"{full}: sha256 mismatch")
        L = meta["leaves"]
        a = np.frombuffer(raw, dtype="<u8")
        return a[:L].view("<i8"), a[L : 2 * L]
    gpath = os.path.join(ROOT, "tests", "golden", f"c{cfg}.json")
    if os.path.exists(gpath):
        g = json.load(open(gpath))
        return np.asarray(g["seeds"], dtype=np.int64), np.asarray(g["fbits"], dtype=np.uint64)
    return None, None


def bench_leaf(cfg, args, dev, sms, rank, world, int_peak):
    """Leaf-search-only configs (BASELINE configs C1/C3/C5): leaf seeds tested/s.
    At N > 1 rank r searches the contiguous leaf range [L r/N, L (r+1)/N) (no
    exchange); seeds tested are summed and the time is the max over ranks.
    Every leaf is checked against the reference's seeds and f bits."""
    from paper_2308_09561_b200 import workloads as W
    from paper_2308_09561_b200._kernels import kernels as K

    spec = W.LEAF_CONFIGS[cfg]
    L_all, n = spec["leaves"], spec["n"]
    # N > 1 and the stealing kernel (n > 24): one cross-GPU leaf queue, every
    # rank holds all leaves (dist.SharedLeafQueue); else contiguous ranges
    shared = world > 1 and n > 24 and os.environ.get("SHK_LEAF_SHARED", "1") != "0"
    l0, l1 = (0, L_all) if shared else ((L_all * rank) // world, (L_all * (rank + 1)) // world)
    L = l1 - l0
    if cfg == 5:
        fp = np.random.default_rng(5).integers(0, 2**64, (L_all, n, 2), dtype=np.uint64)[l0:l1]
        d_hi = dev.DeviceBuffer.from_host(np.ascontiguousarray(fp[..., 0]).ravel())
        d_lo = dev.DeviceBuffer.from_host(np.ascontiguousarray(fp[..., 1]).ravel())
    else:
        k = W.raw_keys(cfg, L_all * n)[l0 * n : l1 * n]
        d_blob = dev.DeviceBuffer.from_host(np.frombuffer(np.ascontiguousarray(k, dtype="<u8").tobytes(), np.uint8))
        d_hi = dev.DeviceBuffer(8 * L * n)
        d_lo = dev.DeviceBuffer(8 * L * n)
        dev.blake2b_fixed_device(d_blob, 8, L * n, 0, d_hi, d_lo)
        d_blob.free()
    d_off = dev.DeviceBuffer.from_host(np.arange(0, (L + 1) * n, n, dtype=np.int64))
    d_seed = dev.DeviceBuffer(8 * L)
    d_fb = dev.DeviceBuffer(8 * L)
    reps = 1 if cfg == 5 else max(1, args.leaf_reps)
    if shared:
        from paper_2308_09561_b200 import dist as shdist

        with shdist.SharedLeafQueue(coll_device()) as q:
            if cfg != 5:
                q.search(d_hi.ptr, d_lo.ptr, d_off.ptr, L, d_seed.ptr, d_fb.ptr)  # warm-up
            ms = sum(q.search(d_hi.ptr, d_lo.ptr, d_off.ptr, L, d_seed.ptr, d_fb.ptr) for _ in range(reps)) / reps
            ms = max_over_ranks(ms, world)
            mine = int((d_seed.download(np.int64, L) >= -1).sum())
            seeds, fbits = q.combine(d_seed.download(np.int64, L), d_fb.download(np.uint64, L))
        per_rank = [int(x) for x in gather_ints(mine, world)]
        seeds_tested = float((seeds + 1).sum())
    else:
        run = lambda: K.leaf_search_device(d_hi.ptr, d_lo.ptr, d_off.ptr, L, 0, d_seed.ptr, d_fb.ptr)
        if cfg != 5:
            run()  # warm-up
        dev.sync()
        barrier(world)
        with dev.timer() as tm:
            for _ in range(reps):
                run()
        ms = max_over_ranks(tm.ms / reps, world)
        seeds = d_seed.download(np.int64, L)
        fbits = d_fb.download(np.uint64, L)
        seeds_tested = reduce_over_ranks(float((seeds + 1).sum()), world, "sum")
        per_rank = None
    w_key = 50 if n <= 32 else 53
    ops = seeds_tested * (n * w_key + W_SEED)
    peak = INT_OPS_PER_CLK_SM * sms * world * MAX_MHZ * 1e6 / 1e12
    ach = ops / (ms * 1e-3) / 1e12
    mean = seeds_tested / L_all
    how = (f", {world} GPUs x one shared leaf queue (CUDA IPC counter)" if shared else
           f", {world} GPUs x contiguous leaf ranges" if world > 1 else "")
    res = {"config": f"C{cfg}: {L_all} leaves x n={n}, plain" + how,
           "kernel": "leaf_steal_kernel (seed-block work stealing)" if n > 24 else "leaf_kernel (fixed teams)",
           "seeds_tested": int(seeds_tested),
           "mean_seeds_per_leaf": round(mean, 1), "ms": round(ms, 3),
           "value": round(seeds_tested / (ms * 1e-3), 1), "unit": "leaf seeds tested/s",
           "roofline": {"bound": "int32-issue", "achieved": round(ach, 3),
                        "peak": round(peak, 2), "unit": "Tops/s", "frac": round(ach / peak, 4),
                        "frac_of_measured": round(ach / (int_peak["measured_best_Tops"] * world), 4),
                        "work": f"(seed+1) x (n x {w_key} + {W_SEED}) int32 ops"}}
    if per_rank is not None:
        res["leaves_solved_per_rank"] = per_rank
    if cfg == 3:
        res["mean_vs_models"] = {"measured": round(mean, 1), "paper_fig2": C3_FIG2_MEAN, "rice_model": C3_RICE_MODEL,
                                 "theorem_4_5_bound": 28200}
    gs, gf = leaf_golden(cfg)
    if gs is not None:
        a, z = l0, min(l1, len(gs))  # the golden leaves inside this rank's range
        if shared and rank != 0:  # every rank holds the combined result: rank 0 checks it
            z = a
        kk = max(0, z - a)
        bad_s = int((seeds[:kk] != gs[a:z]).sum()) if kk else 0
        bad_f = int((fbits[:kk] != gf[a:z]).sum()) if kk else 0
        checked = reduce_over_ranks(kk, world, "sum")
        bad_s = reduce_over_ranks(bad_s, world, "sum")
        bad_f = reduce_over_ranks(bad_f, world, "sum")
        res["parity"] = {"leaves_checked": int(checked), "of_leaves": L_all,
                         "golden": "full population" if len(gs) == L_all else "prefix sample",
                         "seed_mismatches": int(bad_s), "fbits_mismatches": int(bad_f),
                         "seeds_match_reference": bad_s == 0, "fbits_match_reference": bad_f == 0}
    for b_ in (d_hi, d_lo, d_off, d_seed, d_fb):
        b_.free()
    return res


def bench_c2(args, dev, rank):
    """C2 (configs[1]): N=1e5, n=24, b=500 rotate build from resident codes and
    end to end from the host key blob, then its 1e6 queries; parity against
    the reference's descriptor bytes and query outputs (single GPU, rank 0)."""
    from paper_2308_09561_b200 import recsplit
    from paper_2308_09561_b200 import workloads as W

    N, n, b = CFG2["N"], CFG2["n"], CFG2["b"]
    k = W.build_keys(2)
    blob = np.frombuffer(np.ascontiguousarray(k, dtype="<u8").tobytes(), dtype=np.uint8)
    d_blob = dev.DeviceBuffer.from_host(blob)
    d_hi, d_lo = dev.DeviceBuffer(8 * N), dev.DeviceBuffer(8 * N)
    dev.blake2b_fixed_device(d_blob, 8, N, 0, d_hi, d_lo)
    d_blob.free()
    for _ in range(3):
        desc = recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, b, n, CFG2["mode"])
    reps = 10
    dev.sync()
    with dev.timer() as tm:
        for _ in range(reps):
            desc = recsplit.build_hashed_device(d_hi.ptr, d_lo.ptr, N, b, n, CFG2["mode"])
    ms = tm.ms / reps
    pinned_blob = blob.copy()
    recsplit.build_blob(pinned_blob, 8, b, n, CFG2["mode"]).serialize()
    t = time.perf_counter()
    for _ in range(reps):
        out = recsplit.build_blob(pinned_blob, 8, b, n, CFG2["mode"]).serialize()
    e2e_s = (time.perf_counter() - t) / reps
    res = {"config": "C2: ShockHash-RS build N=100,000, n=24, b=500, rotate, eps=0.05",
           "value": round(N / (ms * 1e-3), 1), "unit": "keys/s", "ms": round(ms, 3),
           "e2e": {"value": round(N / e2e_s, 1), "unit": "keys/s", "ms": round(e2e_s * 1e3, 3),
                   "path": "recsplit.build_blob(host blob) -> serialize()"}}
    # 1e6 queries
    idx = W.query_indices(2)
    Q = len(idx)
    qblob = np.frombuffer(np.ascontiguousarray(k[idx], dtype="<u8").tobytes(), dtype=np.uint8)
    d_qb = dev.DeviceBuffer.from_host(qblob)
    d_qhi, d_qlo, d_out = dev.DeviceBuffer(8 * Q), dev.DeviceBuffer(8 * Q), dev.DeviceBuffer(8 * Q)
    dev.blake2b_fixed_device(d_qb, 8, Q, desc.salt, d_qhi, d_qlo)
    dd = desc.device()
    dd.query_device(d_qhi.ptr, d_qlo.ptr, Q, d_out.ptr)
    dev.sync()
    with dev.timer() as tq:
        for _ in range(reps):
            dd.query_device(d_qhi.ptr, d_qlo.ptr, Q, d_out.ptr)
    qms = tq.ms / reps
    res["query"] = {"queries": Q, "value": round(Q / (qms * 1e-3), 1), "unit": "queries/s", "ms": round(qms, 4)}
    qout = d_out.download(np.uint64, Q)
    gpath = os.path.join(ROOT, "tests", "golden", "c2.json")
    if os.path.exists(gpath):
        g = json.load(open(gpath))
        res["parity"] = {"desc_matches_reference": hashlib.sha256(out).hexdigest() == g["desc_sha"],
                         "queries_match_reference": hashlib.sha256(qout.astype("<u8").tobytes()).hexdigest()
                         == g["query_sha"],
                         "bits_per_key": round(len(out) * 8 / N, 6)}
    for b_ in (d_hi, d_lo, d_qb, d_qhi, d_qlo, d_out):
        b_.free()
    return res


def run_reference(args):
    rank, world, local = dist_info()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import refbuild

    r = refbuild.time_build_sample(seconds_target=args.cpu_seconds, steps=args.steps, warmup=args.warmup)
    line = {
        "impl": "reference",
        "metric": "keys/s MPHF build (ShockHash-RS, N=1e7, n=40, b=2000, rotate)",
        "value": r["value"],
        "unit": "keys/s",
        "n_gpus": max(world, args.gpus),
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": r["ms_per_step"],
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic: default_rng(4) uniform 64-bit keys (bounded sample of the C4 workload)",
        "config": {"workload": "C4: ShockHash-RS build N=10,000,000, leaf n=40, bucket b=2000, mode rotate, eps=0.05",
                   "N": CFG["N"], "n": CFG["n"], "b": CFG["b"], "parallelism": "host cores over buckets"},
        "cpu_baseline": {"value": r["value"], "unit": "keys/s", "cores": r["cores"], "kind": r["kind"],
                         "sample": r["sample"]},
        "e2e": {"value": r["value"], "unit": "keys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def relaunch(nproc):
    """`--gpus N` without a launcher: re-run this script under
    torch.distributed.run with N ranks (127.0.0.1 rendezvous)."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    log("bench.py: launching", nproc, "ranks:", " ".join(cmd))
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "4")
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--queries", type=int, default=CFG["queries"])
    ap.add_argument("--query-reps", type=int, default=3)
    ap.add_argument("--check", action="store_true", default=True)
    ap.add_argument("--no-check", dest="check", action="store_false")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu-leaf", action="store_true", help="skip the reference leaf-search CPU baselines")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--leaf-configs", default="1,3,5", help="leaf-search-only configs to add (C1,C3,C5; C5 is one ~12 s launch)")
    ap.add_argument("--leaf-reps", type=int, default=3)
    ap.add_argument("--no-c2", dest="c2", action="store_false", help="skip the C2 build + queries line")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 1)
    rank, world, _ = dist_info()
    if args.impl == "reference":
        run_reference(args)
        return 0
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args.gpus)
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        log(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; reporting the launcher's world size")
    run_ours(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
