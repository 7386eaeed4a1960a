"""SURVEY.md §8(d) "Oracle timing": the CPU oracle as it stands, on the GPU box's host cores,
for every BASELINE row shape, in two modes -- 1 thread (the plain oracle) and all cores (the
same gather loop under OpenMP over batch rows; the qsort permutation is single-threaded in
both).  Also the oracle's propagation (Eq. 2) on the config-1 graph and one hop on a
products-sized graph.  One JSON line per measurement; test/bench infrastructure only.

Bounded samples (stated in each line):
  * tiny, products: full epochs (products' gather over 64 of 299 batches, extrapolated by rows);
  * papers100M / IGB-large / MAG240M shapes: the permutation over the config's real N
    (chunked: U = ceil(N / c) units) or over N' when the RR key sort of all N would dominate the
    run (then scaled by N log N), and the gather of 64 (IGB: 16) batches from a host store of N'
    rows (positions map to rows v mod N'), extrapolated to the epoch by rows.
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402

CORES = os.cpu_count() or 1
SEED, DATA_SEED = 250413266, 2504

SHAPES = [
    # name, N, H, F, B, chunk, store dtype, out dtype, N' (host rows), batches sampled
    ("tiny", 2708, 4, 128, 256, 1, oracle.F32, oracle.BF16, 2708, None),
    ("products", 2_449_029, 4, 100, 8192, 1, oracle.F32, oracle.BF16, 2_449_029, 64),
    ("papers100M", 111_059_956, 4, 128, 8192, 8192, oracle.F32, oracle.BF16, 10_000_000, 64),
    ("igb-large", 100_000_000, 3, 1024, 4096, 1, oracle.F32, oracle.BF16, 2_000_000, 16),
    ("mag240m", 244_160_499, 4, 768, 8192, 1, oracle.F16, oracle.F16, 4_000_000, 64),
]
PERM_FULL_MAX = 10_000_000  # RR sorts of more units than this are timed on N' and scaled by N log N


def emit(d):
    print(json.dumps(d), flush=True)


def time_shape(name, N, H, F, B, chunk, in_dt, out_dt, Np, nb):
    store = oracle.gen_rows(DATA_SEED, in_dt, H, F, np.arange(Np), nthreads=CORES)  # untimed
    U = (N + chunk - 1) // chunk
    if U <= PERM_FULL_MAX:
        t0 = time.perf_counter()
        order = oracle.epoch_order(SEED, N, chunk)
        perm_s = time.perf_counter() - t0
        perm_note = f"full permutation of U = {U} units"
    else:
        t0 = time.perf_counter()
        order = oracle.epoch_order(SEED, Np, chunk)
        perm_np = time.perf_counter() - t0
        perm_s = perm_np * (U * math.log(U)) / (Np * math.log(Np))
        perm_note = f"permutation of N' = {Np} units, scaled by N log N to U = {U}"
    order = order % Np if N > Np else order
    steps = oracle.num_steps(N, B)
    nb = steps if nb is None else min(nb, steps)
    for threads in (1, CORES):
        rows = 0
        t0 = time.perf_counter()
        for t in range(nb):
            s, e = oracle.batch_range(order.shape[0], B, 1, t, 0)
            oracle.gather_cast(store, in_dt, F, H * F, H, F, order[s:e], out_dt, nthreads=threads)
            rows += e - s
        g_s = time.perf_counter() - t0
        epoch_s = perm_s + g_s * (N / rows)
        emit({"kind": "oracle_loader", "shape": name, "threads": threads, "N": N, "host_rows": Np,
              "batches_timed": nb, "permute_s": perm_s, "gather_s": g_s, "epoch_s_extrapolated": epoch_s,
              "nodes_per_s": N / epoch_s,
              "gather_GBs": rows * H * F * ((4 if in_dt == oracle.F32 else 2) + 2) / g_s / 1e9,
              "sample": f"{perm_note}; gather of {nb} of {steps} batches ({rows} rows), epoch by rows"})
    del store


def time_propagation():
    # config 1: the oracle builds the hop tensor itself (CSR, weights, K = 3 SpMMs)
    t0 = time.perf_counter()
    oracle.tiny_hops()
    emit({"kind": "oracle_propagation", "graph": "config-1 (n = 2708, m = 5429, F = 128, K = 3)",
          "threads": 1, "seconds": time.perf_counter() - t0})
    # one hop on a products-sized Erdos-Renyi graph (the GPU bench's shape, numpy RNG)
    n, m, F = 2_449_029, 61_859_140, 100
    rng = np.random.default_rng(DATA_SEED)
    src, dst = rng.integers(0, n, m), rng.integers(0, n, m)
    t0 = time.perf_counter()
    rp, ci = oracle.build_csr(n, src, dst)
    val = oracle.operator_values(n, rp, ci)
    prep_s = time.perf_counter() - t0
    X = rng.standard_normal((n, F)).astype(np.float32)
    t0 = time.perf_counter()
    oracle.spmm(n, rp, ci, val, X)
    hop_s = time.perf_counter() - t0
    emit({"kind": "oracle_propagation", "graph": "products-sized ER (n = 2,449,029, 61.9 M drawn edges)",
          "nnz": int(rp[-1]), "F": F, "threads": 1, "csr_and_weights_s": prep_s, "seconds_per_hop": hop_s,
          "K3_seconds_extrapolated": prep_s + 3 * hop_s})


if __name__ == "__main__":
    emit({"kind": "host", "cores": CORES, "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0]
          .strip(" :\t") if os.path.exists("/proc/cpuinfo") else "?"})
    for shp in SHAPES:
        time_shape(*shp)
    time_propagation()
