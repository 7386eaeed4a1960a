"""Benchmark of the PP-GNN mini-batch loading hot path (arXiv 2504.13266) on B200.

A "step" is one epoch of the whole hot path: pp_epoch_permute
(SGD-RR Philox argsort; the next epoch's order is prefetched on a side stream so it
overlaps this epoch's batches) + every batch of the epoch assembled with the fused
fp32 -> bf16 cast, k batches per pp_next_batches launch (default k = 8, an 8-slot
prefetch ring; k = 1 is one pp_next_batch call per batch, also reported).
value = nodes/s.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--chunk c]
                  [--per-call k]  (k batches per pp_next_batches launch; 1 = pp_next_batch)

N = 1: ogbn-products-shaped (BASELINE configs[1]): N = 2,449,029, F = 100, K = 3 (H = 4),
B = 8192, HBM-resident fp32 hop features (synthetic, §8(d) generator G), bf16 batches.
Secondary keys at N = 1 (each measured after the headline, in its own subprocess where
noted): per_batch_call, gather_only, consumer_fused_linear (§8(f)-1), e2e (host-resident
store over PCIe), double_buffer (§8(a) A6, subprocess), next_rows (§8(f)-2 propagation,
§8(f)-3 storage tier, papers100M compact store; subprocesses), cpu_baseline (the oracle).

N > 1 (torchrun): ogbn-papers100M-shaped (configs[2]): N = 111,059,956, F = 128, K = 3,
B = 8192 per rank, chunk reshuffle c = 8192, nodes sharded round-robin over the ranks,
rows read from the owners' HBM by NVLink peer loads (CUDA IPC).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "batch-assembly nodes/sec"
UNIT = "nodes/s"
SEED0 = 250413266
DATA_SEED = 2504

CONFIGS = {
    "products": dict(N=2_449_029, H=4, F=100, B=8192, chunk=1),
    "papers100M": dict(N=111_059_956, H=4, F=128, B=8192, chunk=8192),
    "tiny": dict(N=2708, H=4, F=128, B=256, chunk=1),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML every ~2 ms (the timed
    region of a products run is only tens of ms), nvidia-smi every 100 ms if NVML is unavailable."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, set of reason names)
        self._stop = threading.Event()
        self._t = None
        self.source = "nvml"
        self._nvml = None
        try:  # initialise NVML before the timed region starts (nvmlInit takes tens of ms)
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(max(0, index))
            self._nvml = (pynvml, h, pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nvml = None

    def _run_nvml(self):
        if self._nvml is None:
            raise RuntimeError("NVML unavailable")
        pynvml, h, mx = self._nvml
        bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
        try:
            while True:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((float(sm), float(mx), {n for n, bit in zip(self.NAMES, bits) if r & bit}))
                if self._stop.wait(0.002):
                    break
        finally:
            pynvml.nvmlShutdown()

    def _run_smi(self):
        self.source = "nvidia-smi"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    r = [x.strip() for x in line.split(",")]
                    if r[0].replace(".", "").isdigit():
                        self.rows.append((float(r[0]), float(r[1]),
                                          {self.NAMES[i] for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"}))
            except Exception:
                pass
            self._stop.wait(0.1)

    def _run(self):
        try:
            self._run_nvml()
        except Exception:
            if not self._stop.is_set():
                self._run_smi()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted(set().union(*(r[2] for r in self.rows))), "samples": len(self.rows),
                "source": self.source}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def committed_traffic(name: str):
    """dram read+write bytes per launch of the dominant kernel from a committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get(name)
    return None


# --------------------------------------------------------------------------- CPU oracle (baseline / reference arm)
def oracle_epoch_sample(cfg, nbatches: int, nthreads: int):
    """The oracle as it stands: permutation of all N units (qsort, 1 thread) + gather+cast of
    the first `nbatches` batches from a host store regenerated with the oracle generator (all rows,
    untimed).  Returns (extrapolated epoch seconds, timings)."""
    import numpy as np

    import oracle

    N, H, F, B, chunk = cfg["N"], cfg["H"], cfg["F"], cfg["B"], cfg["chunk"]
    store = oracle.gen_rows(DATA_SEED, oracle.F32, H, F, np.arange(N), nthreads=nthreads)  # [N, H, F] node-major
    t0 = time.perf_counter()
    order = oracle.epoch_order(SEED0, N, chunk)
    t1 = time.perf_counter()
    steps = oracle.num_steps(N, B)
    nb = min(nbatches, steps)
    rows_done = 0
    for t in range(nb):
        s, e = oracle.batch_range(N, B, 1, t, 0)
        oracle.gather_cast(store, oracle.F32, F, H * F, H, F, order[s:e], oracle.BF16, nthreads=nthreads)
        rows_done += e - s
    t2 = time.perf_counter()
    epoch_s = (t1 - t0) + (t2 - t1) * (N / rows_done)
    return epoch_s, {"permute_s": t1 - t0, "gather_s": t2 - t1, "gather_rows": rows_done, "batches": nb}


def run_reference(args):
    """--impl reference: the CPU oracle (this tier has no runnable reference code)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS["products"]
    nthreads = os.cpu_count() or 1
    times = []
    info = None
    for i in range(args.warmup + args.steps):
        s, info = oracle_epoch_sample(cfg, 16, nthreads)
        if i >= args.warmup:
            times.append(s)
    ms = statistics.median(times) * 1e3
    value = cfg["N"] / (ms / 1e3)
    sample = (f"per step: full-N permutation + gather+cast of {info['batches']} of 299 batches "
              f"({info['gather_rows']} rows), epoch time extrapolated by rows")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32->bf16", "data": "synthetic",
        "config": config_dict("products", cfg, 1, "none (host)"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def config_dict(name, cfg, W, l2):
    return {"workload": f"{name}-shaped", "num_nodes": cfg["N"], "feat_dim": cfg["F"], "hops_K": cfg["H"] - 1,
            "batch_size": cfg["B"], "chunk": cfg["chunk"], "store": "fp32 node-major, HBM-resident",
            "out": "bf16", "world_size": W, "l2_policy": l2}


# --------------------------------------------------------------------------- GPU arm
def epoch_loop(L, seed, next_seed, chunk, steps, slots, slot_bytes, k, stream, node_slots=None, ev_mid=None):
    """One timed step: pp_epoch_permute(seed) (switches to the prefetched order when the previous
    epoch prefetched it), pp_epoch_prefetch(next_seed) on the side stream, then every batch of the
    epoch, k per pp_next_batches launch (k = 1: pp_next_batch), into consecutive slots of the ring
    (a call never wraps it).  tests/test_gpu_timed_path.py runs this exact loop against the oracle."""
    L.epoch_permute(seed, chunk, stream)
    if next_seed is not None:
        L.epoch_prefetch(next_seed, chunk)  # next epoch's order overlaps this epoch's batches
    if ev_mid is not None:
        ev_mid.record(stream)
    nslots = len(slots)
    done = 0
    while done < steps:
        s0 = done % nslots
        nodes = None if node_slots is None else node_slots[s0]
        if k == 1:
            L.next_batch(slots[s0], None, nodes, stream)
            done += 1
        else:
            n = min(k, steps - done, nslots - s0)
            done += len(L.next_batches(n, slots[s0], slot_bytes, None, nodes, stream))


def ring_slots(steps, per_call, slot_bytes):
    """Output ring of the timed loop: one slot per step of the epoch, capped at 4 GB (>= 1 GB >> L2,
    so the outputs go to DRAM)."""
    return min(steps, max(per_call, int(4e9 // slot_bytes)))


def run_ours(args):
    import torch

    import paper_2504_13266_b200 as pp

    W = args.gpus
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    shared_gpu = W > ndev  # path check with several ranks per GPU (e.g. on a 1-GPU box): gloo plumbing
    local = local % ndev
    torch.cuda.set_device(local)
    dist = None
    if W > 1:
        import torch.distributed as dist

        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    name = args.config or ("products" if W == 1 else "papers100M")
    cfg = dict(CONFIGS[name])
    if args.chunk is not None:
        cfg["chunk"] = args.chunk
    N, H, F, B, chunk = cfg["N"], cfg["H"], cfg["F"], cfg["B"], cfg["chunk"]
    stream = torch.cuda.Stream()

    desc = dict(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16,
                device=local)
    if W > 1:
        desc.update(world_size=W, rank=rank, peers=pp.PP_PEERS_IPC)
    L = pp.Loader(**desc)
    L.fill_synthetic(DATA_SEED)
    if W > 1:
        h = pp.pp_export_store(L.h)
        hs = [None] * W
        dist.all_gather_object(hs, h)
        pp.pp_import_peer_stores(L.h, b"".join(hs))
    L.set_stream(stream)
    info = L.query()
    steps = info["steps_per_epoch"]
    rec_in, rec_out = info["record_bytes_in"], info["record_bytes_out"]

    slot_bytes = B * H * F * 2
    nslots = ring_slots(steps, args.per_call, slot_bytes)
    ring = torch.empty((nslots, B, H, F), dtype=torch.bfloat16, device="cuda")
    slots = list(ring.unbind(0))  # slot views made once, not per call (torch indexing costs ~1 us)
    # rows this rank assembles per epoch (for the algorithmic bytes)
    my_rows = sum(max(0, min(B, N - (t * W * B + rank * B))) for t in range(steps))
    U = -(-N // chunk)
    # kernels of ours per permutation: one-CTA sort (U <= 4096) or the 6-kernel bucket sort
    # (+ ragged-chunk search), + the chunk expansion when chunk > 1
    perm_kernels = (1 if U <= 4096 else 6 + (chunk > 1)) + (chunk > 1)

    def timed(k, nsteps, sampler_index=None):
        def epoch(e, ev_mid=None):
            epoch_loop(L, SEED0 + e, SEED0 + e + 1 if args.prefetch else None, chunk, steps, slots, slot_bytes, k,
                       stream, ev_mid=ev_mid)

        with torch.cuda.stream(stream):
            for e in range(args.warmup):
                epoch(e)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        evs = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(nsteps)]
        clk = ClockSampler(sampler_index) if sampler_index is not None else None
        if clk is not None:
            clk.__enter__()
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            start.record(stream)
            for i in range(nsteps):
                evs[i][0].record(stream)
                epoch(args.warmup + i, evs[i][1])
                evs[i][2].record(stream)
            end.record(stream)
        torch.cuda.synchronize()
        if clk is not None:
            clk.__exit__(None, None, None)
        if dist:
            dist.barrier()
        t = [start.elapsed_time(end), sum(b.elapsed_time(c) for _, b, c in evs),
             sum(a.elapsed_time(b) for a, b, _ in evs)]
        if dist:
            tt = torch.tensor(t, device="cpu" if shared_gpu else "cuda", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = tt.tolist()
        launches, done = 0, 0  # gather launches per epoch (calls never wrap the ring)
        while done < steps:
            done += 1 if k == 1 else min(k, steps - done, nslots - done % nslots)
            launches += 1
        per_launch_ms = t[1] / (nsteps * launches)
        bytes_per_launch = my_rows * (rec_in + rec_out + 4) / launches
        return {"total_ms": t[0], "gather_ms": t[1], "perm_ms": t[2], "per_launch_ms": per_launch_ms,
                "bytes_per_launch": bytes_per_launch, "achieved": bytes_per_launch / (per_launch_ms / 1e3) / 1e9,
                "launches": launches, "clocks": clk.summary() if clk is not None else None}

    k = max(1, args.per_call)
    m = timed(k, args.steps, sampler_index=local)
    ms_per_step = m["total_ms"] / args.steps
    value = N * args.steps / (m["total_ms"] / 1e3)  # all ranks together assemble N rows per epoch
    peak, peak_kind = peaks()
    if W == 1:
        roofline = {"bound": "hbm", "achieved": m["achieved"], "peak": peak, "unit": "GB/s",
                    "frac": m["achieved"] / peak, "traffic": committed_traffic(f"gather_{name}_k{k}"),
                    "kernel": "k_gather_vec<bf16>", "peak_kind": peak_kind,
                    "algorithmic_bytes_per_node": rec_in + rec_out + 4,
                    "frac_of_8TBs_nominal": m["achieved"] / 8000.0}
    else:
        # pull design: (W-1)/W of each rank's rows arrive over NVLink, read from the owner's
        # exchange copy (already cast: rec_out bytes) or, without one, as fp32 records (rec_in)
        rec_nvl = rec_out if L.query()["exchange_cast"] else rec_in
        nvl = m["bytes_per_launch"] / (rec_in + rec_out + 4) * rec_nvl * (W - 1) / W
        achieved = nvl / (m["per_launch_ms"] / 1e3) / 1e9
        roofline = {"bound": "nvlink", "achieved": achieved, "peak": 770.0, "unit": "GB/s", "frac": achieved / 770.0,
                    "traffic": None, "kernel": "k_gather_tma<bf16, sharded>",
                    "peak_kind": "guide-measured peer copy per direction (B200_PROFILING.md)",
                    "algorithmic_nvlink_bytes_per_node": rec_nvl * (W - 1) / W, "hbm_GBs": m["achieved"],
                    "exchange_cast": bool(L.query()["exchange_cast"])}
    roofline.update({"per_launch_us": m["per_launch_ms"] * 1e3, "algorithmic_bytes_per_launch": m["bytes_per_launch"],
                     "note": "per-launch time = CUDA-event span from the epoch's first gather to its last / launches "
                             "(includes launch gaps and the overlapped next-epoch permutation)"})
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": W, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak" if W == 1 else "strong",
        "vs_baseline": None, "dtype": "f32->bf16", "data": "synthetic (§8(d) generator G, filled in place)",
        "config": config_dict(name, cfg, W, "inputs > L2 (3.9 GB store), outputs rotate over a "
                                            f"{ring.numel() * 2 / 1e9:.2f} GB ring of {nslots} slots"),
        "roofline": roofline, "gpu_launches": (perm_kernels + m["launches"]) * args.steps, "clocks": m["clocks"],
        "batches_per_launch": k, "prefetch_next_epoch_order": bool(args.prefetch),
        # SURVEY.md §8(d) timing protocol: (a) gather-only nodes/s (span of the epoch's gathers),
        # (b) whole epochs incl. the permutation (= value), (c) per-call latency (per_batch_call)
        "gather_only": {"value": N * args.steps / (m["gather_ms"] / 1e3), "unit": UNIT,
                        "ms_per_epoch": m["gather_ms"] / args.steps},
    }
    if k != 1 and not args.skip_k1:
        m1 = timed(1, max(3, args.steps // 2))
        result["per_batch_call"] = {
            "value": N * max(3, args.steps // 2) / (m1["total_ms"] / 1e3), "unit": UNIT,
            "ms_per_step": m1["total_ms"] / max(3, args.steps // 2), "achieved_GBs": m1["achieved"],
            "per_call_us": m1["total_ms"] * 1e3 / (max(3, args.steps // 2) * steps),
            "note": "one pp_next_batch call (one launch) per batch from Python (Loader.next_batch fast path)"}
    del ring, slots
    torch.cuda.synchronize()
    if dist:
        dist.barrier()  # peers read this rank's store until every rank is done
    L.close()
    torch.cuda.empty_cache()

    if W > 1 and not args.skip_weak:
        # Weak-scaling companion of the N = 1 headline: a products-shaped shard per rank
        # (N_total = 2,449,029 x W), one global permutation, (W-1)/W of every batch read from
        # peers -- the per-GPU work of the single-GPU line, so the two compare directly.
        N = CONFIGS["products"]["N"] * W
        H, F, B, chunk = CONFIGS["products"]["H"], CONFIGS["products"]["F"], CONFIGS["products"]["B"], 1
        L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16,
                      device=local, world_size=W, rank=rank, peers=pp.PP_PEERS_IPC)
        L.fill_synthetic(DATA_SEED)
        hs = [None] * W
        dist.all_gather_object(hs, pp.pp_export_store(L.h))
        pp.pp_import_peer_stores(L.h, b"".join(hs))
        L.set_stream(stream)
        info = L.query()
        steps = info["steps_per_epoch"]
        rec_in, rec_out = info["record_bytes_in"], info["record_bytes_out"]
        slot_bytes = B * H * F * 2
        nslots = min(steps, max(args.per_call, int(4e9 // slot_bytes)))
        ring = torch.empty((nslots, B, H, F), dtype=torch.bfloat16, device="cuda")
        slots = list(ring.unbind(0))
        my_rows = sum(max(0, min(B, N - (t * W * B + rank * B))) for t in range(steps))
        mw = timed(k, args.steps)
        result["weak_products"] = {
            "value": N * args.steps / (mw["total_ms"] / 1e3), "unit": UNIT, "num_nodes": N,
            "ms_per_step": mw["total_ms"] / args.steps, "per_gpu_nodes_per_s": N * args.steps / (mw["total_ms"] / 1e3) / W,
            "exchange_cast": bool(info["exchange_cast"]),
            "note": "products-shaped shard per rank, global permutation, peer reads; same per-GPU work as N = 1"}
        del ring, slots
        torch.cuda.synchronize()
        dist.barrier()
        L.close()
        torch.cuda.empty_cache()

    if W == 1 and name == "products" and not args.skip_consumer:
        result["consumer_fused_linear"] = consumer_fused_linear(pp, torch, cfg, args)
    if W == 1 and not args.skip_e2e:
        result["e2e"] = e2e_host_store(pp, torch, cfg, args)
    if W == 1 and name == "products" and not args.skip_double_buffer:
        result["double_buffer"] = double_buffer_secondary()
    if W == 1 and name == "products" and not args.skip_next_rows:
        result["next_rows"] = next_rows_secondary()
    if rank == 0 and W == 1 and not args.skip_cpu:
        nthreads = os.cpu_count() or 1
        s, inf = oracle_epoch_sample(cfg, 32, nthreads)
        result["cpu_baseline"] = {
            "value": N / s, "unit": UNIT, "cores": nthreads, "kind": "oracle",
            "sample": (f"full-N permutation (1 thread, qsort) + gather+cast of {inf['batches']} batches "
                       f"({inf['gather_rows']} rows, {nthreads} OpenMP threads); epoch extrapolated by rows"),
            "permute_s": inf["permute_s"], "gather_s": inf["gather_s"]}
    if rank == 0:
        print(json.dumps(result))
    if dist:
        dist.destroy_process_group()


def consumer_fused_linear(pp, torch, cfg, args, D=512, k=8, reps=5):
    """§8(f)-1: the batch consumed by SIGN's per-hop linear layer (hidden 512) in
    the fused tcgen05 kernel (pp_next_batches_linear) -- epochs of permutation + fused
    gather/cast/GEMM, the batch never written to HBM.  Bound: HBM (1600 B read + 4096 B of bf16 Z
    written per node); the tensor work is 2*H*F*D = 410 kFLOP per node."""
    import numpy as np

    N, H, F, B = cfg["N"], cfg["H"], cfg["F"], cfg["B"]
    L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16)
    L.fill_synthetic(DATA_SEED)
    st = torch.cuda.Stream()
    L.set_stream(st)
    steps = L.query()["steps_per_epoch"]
    W = torch.from_numpy((np.random.default_rng(0).standard_normal((H, F, D)) / 10).astype(np.float32)).cuda()
    W = W.to(torch.bfloat16)
    nslots = steps  # one Z slot per step (10 GB): back-to-back launches may overlap (PDL)
    Z = torch.empty((nslots, B, H, D), dtype=torch.bfloat16, device="cuda")
    zs = B * H * D * 2

    def epoch(e):
        L.epoch_permute(SEED0 + e, cfg["chunk"], st)
        L.epoch_prefetch(SEED0 + e + 1, cfg["chunk"])
        done = 0
        while done < steps:
            s0 = done % nslots
            done += len(L.next_batches_linear(min(k, steps - done, nslots - s0), W, D, Z[s0], "bf16", zs, st))

    with torch.cuda.stream(st):
        epoch(0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        a.record(st)
        for i in range(reps):
            epoch(1 + i)
        b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    L.close()
    del Z
    torch.cuda.empty_cache()
    peak, _ = peaks()
    per_node = H * F * 4 + H * D * 2 + 4
    return {"value": N / (ms / 1e3), "unit": UNIT, "ms_per_step": ms, "hidden": D,
            "achieved_GBs": N * per_node / ms / 1e6, "frac_hbm": N * per_node / ms / 1e6 / peak,
            "tflops": 2.0 * N * H * F * D / ms / 1e9,
            "note": "fused gather + cast + per-hop linear (tcgen05, TMEM accumulators); "
                    "unfused loader + cuBLAS reference: profiles/r1e_bench_fused_linear.jsonl"}


def _script_lines(script, env_extra, timeout=600, args=()):
    """Run a scripts/ measurement in a subprocess (own CUDA context); its JSON lines, or an error."""
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", script), *args], env=env, capture_output=True,
                       text=True, timeout=timeout)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    if not lines:
        raise RuntimeError((r.stderr or "no output")[-300:])
    return lines


def next_rows_secondary():
    """The §8(f) rows measured by their scripts: GPU propagation (Eq. (2), products-sized graph),
    the storage tier (hop files, chunk reshuffling) and the paper's papers100M setup (compact
    store of the labelled nodes)."""
    out = {}
    try:
        prop = _script_lines("bench_propagate.py", {}, timeout=240)
        out["propagation"] = {"ms_per_hop": prop[0]["ms_per_hop"], "frac_hbm": prop[0]["frac_hbm"],
                              "into_store_ms_per_hop": prop[-1]["ms_per_hop"], "nnz": prop[0]["nnz"],
                              "note": "bit-identical to the CPU oracle (tests/test_gpu_propagate*.py)"}
    except Exception as e:
        out["propagation"] = {"error": repr(e)[:300]}
    try:
        st = _script_lines("bench_storage.py", {"PP_STORAGE_EPOCHS": "1"}, timeout=300)[-1]
        out["storage_tier"] = {k: st[k] for k in ("chunk", "storage_mode", "nodes_per_s", "storage_GBs",
                                                  "seq_read_GBs_measured", "frac_of_seq_read", "sampled_step_bit_exact")}
    except Exception as e:
        out["storage_tier"] = {"error": repr(e)[:300]}
    try:
        lab = _script_lines("bench_configs.py", {}, timeout=240, args=("papers100M-labelled",))
        out["papers100M_labelled"] = [{k: d[k] for k in ("config", "N", "N_total", "ms_per_epoch", "nodes_per_s", "frac")}
                                      for d in lab]
    except Exception as e:
        out["papers100M_labelled"] = {"error": repr(e)[:300]}
    return out


def double_buffer_secondary():
    """§8(a) A6: the paper's double buffer with a host-resident store and a
    SIGN-style training step (CUDA-graphed) as the consumer -- scripts/bench_double_buffer.py in a
    subprocess (its own CUDA context), summary line only."""
    env = dict(os.environ, DB_GRAPH="1", DB_PLACEMENT="host", DB_CHUNK="1", DB_CTAS="8", DB_EPOCHS="2")
    try:
        r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "bench_double_buffer.py")], env=env,
                           capture_output=True, text=True, timeout=300)
        lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
        modes = {d["mode"]: d["ms_per_epoch"] for d in lines if "mode" in d}
        summ = [d for d in lines if "double_buffer_speedup" in d]
        if not summ:
            return {"error": (r.stderr or "no output")[-300:]}
        return {"speedup": summ[0]["double_buffer_speedup"], "loading_hidden": summ[0]["loader_hidden_fraction"],
                "ms_per_epoch": modes, "store": "pinned host memory (zero-copy, SGD-RR)",
                "consumer": "SIGN-style training step in CUDA graphs", "paper": "1.9x host-resident (PAPER.md:345)"}
    except Exception as e:  # the secondary line must never break the headline
        return {"error": repr(e)[:300]}


def e2e_host_store(pp, torch, cfg, args):
    """Same epoch with the hop store in pinned host memory (the paper's host placement,
    PAPER.md:287-288): every feature byte crosses host->device inside the timed region
    (UVA zero-copy reads), and each batch's node ids are read back to host."""
    N, H, F, B, chunk = cfg["N"], cfg["H"], cfg["F"], cfg["B"], cfg["chunk"]
    L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16,
                  hbm_budget_bytes=-1)
    L.fill_synthetic(DATA_SEED)
    stream = torch.cuda.Stream()
    L.set_stream(stream)
    info = L.query()
    steps = info["steps_per_epoch"]
    out = [torch.empty((B, H, F), dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    nodes = torch.empty((steps, B), dtype=torch.int64, device="cuda")
    host_nodes = torch.empty((steps, B), dtype=torch.int64, pin_memory=True)

    def epoch(e):
        L.epoch_permute(SEED0 + e, chunk, stream)
        for t in range(steps):
            L.next_batch(out[t % 2], None, nodes[t], stream)
        host_nodes.copy_(nodes, non_blocking=True)

    with torch.cuda.stream(stream):
        epoch(0)
    torch.cuda.synchronize()
    reps = 2
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        a.record(stream)
        for i in range(reps):
            epoch(1 + i)
        b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    L.close()
    return {"value": N / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": N * info["record_bytes_in"],
            "d2h_bytes_per_step": N * 8, "ms_per_step": ms,
            "how": "store in pinned host memory, read zero-copy over PCIe by the gather kernel; node ids D2H"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS))
    ap.add_argument("--chunk", type=int, default=None)
    ap.add_argument("--per-call", type=int, default=8,
                    help="batches per pp_next_batches launch (an 8-slot prefetch ring); 1 = pp_next_batch")
    ap.add_argument("--skip-k1", action="store_true", help="skip the secondary one-call-per-batch measurement")
    ap.add_argument("--prefetch", type=int, default=1, help="overlap the next epoch's permutation (1/0)")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-consumer", action="store_true", help="skip the §8(f)-1 fused-linear measurement")
    ap.add_argument("--skip-double-buffer", action="store_true", help="skip the §8(a) A6 double-buffer measurement")
    ap.add_argument("--skip-weak", action="store_true", help="N > 1: skip the products-shaped weak-scaling line")
    ap.add_argument("--skip-next-rows", action="store_true",
                    help="skip the §8(f) propagation / storage-tier / compact-store measurements")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        import __graft_entry__ as ge

        ge.build()
        run_ours(args)


if __name__ == "__main__":
    main()
