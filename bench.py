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

N > 1 (torchrun, one process per GPU): weak scaling of the same per-GPU work -- a products-shaped
shard per rank (N_total = 2,449,029 x N), one global permutation, nodes sharded round-robin, the
(N-1)/N remote rows of every batch read from the owners' HBM by NVLink peer loads (CUDA IPC; the
owners keep cast exchange copies).  Secondary keys at N > 1: exchange_nccl (the same epochs with an
NCCL all-to-all exchange, SURVEY.md §8(e)'s baseline), papers100M (configs[2]: N = 111,059,956,
F = 128, c = 8192, sharded over the N ranks, strong scaling), e2e (every shard in shared pinned host
memory), memory_plan (per rank), nvlink_peer_copy_GBs (the NVLink denominator, measured in the run).
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
def oracle_epoch_sample(cfg, nbatches: int, nthreads: int):  # noqa: D401
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


def ring_plan(steps, per_call, slot_bytes, free_bytes, cap=4e9, reserve=2 << 30):
    """Slots of the timed output ring: one per step of the epoch, at most `cap` bytes and at most the
    HBM left after the store, the exchange copy and the order minus a reserve, but never fewer than
    one launch's worth (per_call slots)."""
    ring_bytes = max(per_call * slot_bytes, min(cap, free_bytes - reserve))
    return int(min(steps, max(per_call, ring_bytes // slot_bytes)))


def ring_slots(steps, per_call, slot_bytes):
    """Output ring of the timed loop: one slot per step of the epoch, capped at 4 GB (>= 1 GB >> L2,
    so the outputs go to DRAM)."""
    return min(steps, max(per_call, int(4e9 // slot_bytes)))


def measure_peer_copy(torch, local, W, shared_gpu):
    """NVLink denominator measured in this run: every rank copies 1 GiB from the next rank's GPU into
    its own (cudaMemcpyPeer through torch, all ranks at once, so every GPU also serves one reader),
    best of 5, CUDA events on the local device."""
    if shared_gpu or W < 2:
        return None
    peer = (local + 1) % W
    src = torch.empty(1 << 30, dtype=torch.uint8, device=f"cuda:{peer}")
    dst = torch.empty(1 << 30, dtype=torch.uint8, device=f"cuda:{local}")
    best = 0.0
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        b.synchronize()
        best = max(best, (1 << 30) / (a.elapsed_time(b) / 1e3) / 1e9)
    del src, dst
    torch.cuda.empty_cache()
    return best


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
    stream = torch.cuda.Stream()
    k = max(1, args.per_call)

    def gather_all(obj):
        if not dist:
            return [obj]
        out = [None] * W
        dist.all_gather_object(out, obj)
        return out

    peer_gbs = measure_peer_copy(torch, local, W, shared_gpu)
    peer_all = gather_all(peer_gbs)
    peer_meas = [x for x in peer_all if x]
    nvl_peak = statistics.median(peer_meas) if peer_meas else 770.0
    nvl_kind = (f"measured in this run: peer copy into each rank from the next one, median over ranks "
                f"{[round(x, 1) for x in peer_meas]}" if peer_meas else
                "fallback: guide-measured peer copy per direction (B200_PROFILING.md), not measurable here")

    def make_loader(cfg, mode="ipc", budget=0):
        desc = dict(num_nodes=cfg["N"], num_hops=cfg["H"], feat_dim=cfg["F"], dtype=pp.PP_F32, batch_size=cfg["B"],
                    out_dtype=pp.PP_BF16, device=local, hbm_budget_bytes=budget)
        uid = None
        if mode == "nccl":
            uid = gather_all(pp.pp_nccl_unique_id() if rank == 0 else None)[0]
            desc.update(peers=pp.PP_PEERS_NCCL, nccl_unique_id=uid, world_size=W, rank=rank)
        elif W > 1:
            desc.update(world_size=W, rank=rank, peers=pp.PP_PEERS_IPC)
        L = pp.Loader(**desc)
        L.fill_synthetic(DATA_SEED)
        if W > 1 and mode == "ipc":
            pp.pp_import_peer_stores(L.h, b"".join(gather_all(pp.pp_export_store(L.h))))
        L.set_stream(stream)
        return L

    def measure(L, cfg, kk, nsteps, sampler_index=None, ring_cap=4e9, label=""):
        """Timed epochs of bench.epoch_loop on loader L: returns the timing dict and the memory plan."""
        N, H, F, B, chunk = cfg["N"], cfg["H"], cfg["F"], cfg["B"], cfg["chunk"]
        info = L.query()
        steps = info["steps_per_epoch"]
        rec_in, rec_out = info["record_bytes_in"], info["record_bytes_out"]
        slot_bytes = B * H * F * 2
        free, total = torch.cuda.mem_get_info()
        nslots = ring_plan(steps, kk, slot_bytes, free, ring_cap)
        ring = torch.empty((nslots, B, H, F), dtype=torch.bfloat16, device="cuda")
        slots = list(ring.unbind(0))  # slot views made once, not per call (torch indexing costs ~1 us)
        my_rows = sum(max(0, min(B, N - (t * W * B + rank * B))) for t in range(steps))
        plan = {"rank": rank, "device": local, "gpu_total": total, "gpu_free_before_ring": free,
                "ring_bytes": nslots * slot_bytes, "ring_slots": nslots,
                **{x: info[x] for x in ("rows_hbm", "rows_spill", "hbm_store_bytes", "hbm_exchange_bytes",
                                        "hbm_scratch_bytes", "host_spill_bytes", "exchange_cast", "all_to_all")}}

        def epoch(e, ev_mid=None):
            epoch_loop(L, SEED0 + e, SEED0 + e + 1 if args.prefetch else None, chunk, steps, slots, slot_bytes, kk,
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
        launches, done = 0, 0  # batch launches per epoch (calls never wrap the ring)
        while done < steps:
            done += 1 if kk == 1 else min(kk, steps - done, nslots - done % nslots)
            launches += 1
        per_launch_ms = t[1] / (nsteps * launches)
        bytes_per_launch = my_rows * (rec_in + rec_out + 4) / launches
        del ring, slots
        return {"total_ms": t[0], "gather_ms": t[1], "perm_ms": t[2], "per_launch_ms": per_launch_ms,
                "bytes_per_launch": bytes_per_launch, "achieved": bytes_per_launch / (per_launch_ms / 1e3) / 1e9,
                "launches": launches, "steps": steps, "nslots": nslots, "my_rows": my_rows, "rec_in": rec_in,
                "rec_out": rec_out, "exchange_cast": info["exchange_cast"], "all_to_all": info["all_to_all"],
                "clocks": clk.summary() if clk is not None else None, "plan": plan}

    def nvlink_roofline(m, kernel):
        # (W-1)/W of each rank's rows come from peers: from the owner's exchange copy (cast: rec_out
        # bytes), its fp32 records (rec_in) without one, or packed + cast by the owner (a2a: rec_out)
        rec_nvl = m["rec_out"] if (m["exchange_cast"] or m["all_to_all"]) else m["rec_in"]
        nvl = m["my_rows"] / m["launches"] * rec_nvl * (W - 1) / W
        achieved = nvl / (m["per_launch_ms"] / 1e3) / 1e9
        return {"bound": "nvlink", "achieved": achieved, "peak": nvl_peak, "unit": "GB/s", "frac": achieved / nvl_peak,
                "traffic": None, "kernel": kernel, "peak_kind": nvl_kind,
                "algorithmic_nvlink_bytes_per_node": rec_nvl * (W - 1) / W, "hbm_GBs": m["achieved"],
                "per_launch_us": m["per_launch_ms"] * 1e3,
                "note": "per-launch time = CUDA-event span of the epoch's batch launches / launches, max over ranks"}

    def finish(L):
        torch.cuda.synchronize()
        if dist:
            dist.barrier()  # peers read this rank's store until every rank is done
        L.close()
        torch.cuda.empty_cache()

    # ---- headline.  N = 1: products-shaped (configs[1]).  N > 1: weak scaling -- a products-shaped
    # shard per rank (N_total = 2,449,029 x W), one global permutation, (W-1)/W of every batch read
    # from the owners' HBM over NVLink (cast exchange copies) -- the per-GPU work of the N = 1 line.
    name = args.config or "products"
    cfg = dict(CONFIGS[name])
    if args.chunk is not None:
        cfg["chunk"] = args.chunk
    if W > 1 and name == "products":
        cfg["N"] = CONFIGS["products"]["N"] * W
    N, chunk = cfg["N"], cfg["chunk"]
    U = -(-N // chunk)
    # kernels of ours per permutation: one-CTA sort (U <= 4096) or the 6-kernel bucket sort
    # (+ ragged-chunk search), + the chunk expansion when chunk > 1
    perm_kernels = (1 if U <= 4096 else 6 + (chunk > 1)) + (chunk > 1)
    L = make_loader(cfg)
    m = measure(L, cfg, k, args.steps, sampler_index=local)
    plans = gather_all(m["plan"])
    ms_per_step = m["total_ms"] / args.steps
    value = N * args.steps / (m["total_ms"] / 1e3)  # all ranks together assemble N rows per epoch
    peak, peak_kind = peaks()
    store_gb = N * m["rec_in"] / 1e9
    if W == 1:
        roofline = {"bound": "hbm", "achieved": m["achieved"], "peak": peak, "unit": "GB/s",
                    "frac": m["achieved"] / peak, "traffic": committed_traffic(f"gather_{name}_k{k}"),
                    "kernel": "k_gather_vec<bf16>", "peak_kind": peak_kind,
                    "algorithmic_bytes_per_node": m["rec_in"] + m["rec_out"] + 4,
                    "frac_of_8TBs_nominal": m["achieved"] / 8000.0, "per_launch_us": m["per_launch_ms"] * 1e3,
                    "algorithmic_bytes_per_launch": m["bytes_per_launch"],
                    "note": "per-launch time = CUDA-event span from the epoch's first gather to its last / launches "
                            "(includes launch gaps and the overlapped next-epoch permutation)"}
    else:
        roofline = nvlink_roofline(m, "k_gather_tma<bf16, sharded> (peer reads)")
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": W, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32->bf16", "data": "synthetic (§8(d) generator G, filled in place)",
        "config": config_dict(name if W == 1 else f"{name}-weak", cfg, W,
                              f"inputs > L2 ({store_gb:.1f} GB store), outputs rotate over a "
                              f"{m['nslots'] * cfg['B'] * cfg['H'] * cfg['F'] * 2 / 1e9:.2f} GB ring of "
                              f"{m['nslots']} slots per rank"),
        "roofline": roofline, "gpu_launches": (perm_kernels + m["launches"]) * args.steps, "clocks": m["clocks"],
        "batches_per_launch": k, "prefetch_next_epoch_order": bool(args.prefetch),
        # SURVEY.md §8(d) timing protocol: (a) gather-only nodes/s (span of the epoch's gathers),
        # (b) whole epochs incl. the permutation (= value), (c) per-call latency (per_batch_call)
        "gather_only": {"value": N * args.steps / (m["gather_ms"] / 1e3), "unit": UNIT,
                        "ms_per_epoch": m["gather_ms"] / args.steps},
        "memory_plan": plans,
    }
    if W > 1:
        result["nvlink_peer_copy_GBs"] = peer_all
    if k != 1 and not args.skip_k1:
        n1 = max(3, args.steps // 2)
        m1 = measure(L, cfg, 1, n1)
        result["per_batch_call"] = {
            "value": N * n1 / (m1["total_ms"] / 1e3), "unit": UNIT, "ms_per_step": m1["total_ms"] / n1,
            "achieved_GBs": m1["achieved"], "per_call_us": m1["total_ms"] * 1e3 / (n1 * m1["steps"]),
            "note": "one pp_next_batch call (one launch) per batch from Python (Loader.next_batch fast path)"}
    finish(L)

    if W > 1 and not args.skip_nccl:
        # SURVEY.md §8(e) baseline on the same workload: every step's rows exchanged by an NCCL
        # all-to-all (owner packs + casts, ncclSend/ncclRecv, receiver unpacks)
        if shared_gpu:
            result["exchange_nccl"] = {"unavailable": "NCCL refuses two ranks on one GPU (path check run)"}
        else:
            try:
                L = make_loader(cfg, mode="nccl")
                mn = measure(L, cfg, k, max(3, args.steps // 2))
                result["exchange_nccl"] = {
                    "value": N * max(3, args.steps // 2) / (mn["total_ms"] / 1e3), "unit": UNIT,
                    "ms_per_step": mn["total_ms"] / max(3, args.steps // 2),
                    "roofline": nvlink_roofline(mn, "pack (k_gather_vec) + ncclSend/ncclRecv + k_a2a_unpack"),
                    "memory_plan": gather_all(mn["plan"])}
                finish(L)
            except Exception as e:  # the baseline must never break the headline
                result["exchange_nccl"] = {"error": repr(e)[:300]}
    if W > 1 and not args.skip_papers and shared_gpu:
        result["papers100M"] = {"unavailable": "needs one GPU per rank (227 GB of shards; path check run)"}
    elif W > 1 and not args.skip_papers:
        # BASELINE configs[2]: papers100M-shaped, c = 8192, sharded over the W ranks (strong scaling)
        pcfg = dict(CONFIGS["papers100M"])
        try:
            L = make_loader(pcfg)
            mp_ = measure(L, pcfg, k, max(3, args.steps // 2))
            result["papers100M"] = {
                "value": pcfg["N"] * max(3, args.steps // 2) / (mp_["total_ms"] / 1e3), "unit": UNIT,
                "ms_per_step": mp_["total_ms"] / max(3, args.steps // 2), "scaling": "strong",
                "config": config_dict("papers100M", pcfg, W, "inputs > L2"),
                "roofline": nvlink_roofline(mp_, "k_gather_tma<bf16, sharded> (peer reads)"),
                "memory_plan": gather_all(mp_["plan"])}
            finish(L)
        except Exception as e:
            result["papers100M"] = {"error": repr(e)[:300]}
    if not args.skip_e2e:
        result["e2e"] = e2e_host_store(pp, torch, CONFIGS["products"], args, W=W, rank=rank, local=local,
                                       gather_all=gather_all, dist=dist, shared_gpu=shared_gpu)
    if W == 1 and name == "products" and not args.skip_consumer:
        result["consumer_fused_linear"] = consumer_fused_linear(pp, torch, cfg, args)
    if W == 1 and name == "products" and not args.skip_double_buffer:
        result["double_buffer"] = double_buffer_secondary()
    if W == 1 and name == "products" and not args.skip_next_rows:
        result["next_rows"] = next_rows_secondary()
    if rank == 0 and W == 1 and not args.skip_cpu:
        result["cpu_baseline"] = cpu_baseline(cfg)
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
            "note": "fused gather + cast + per-hop linear (k_gather_linear_kc: TMA gather4 A chunks, tcgen05 CTA pairs, TMEM accumulators); "
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
        p0 = prop[0]
        out["propagation"] = {"ms_per_hop": p0["ms_per_hop"], "frac_hbm": p0["frac_hbm"],
                              "frac_hbm_basis": "no-reuse bytes (every nonzero reads its neighbour row, column, weight)",
                              "compulsory_bytes_per_hop": p0.get("compulsory_bytes_per_hop"),
                              "compulsory_GBs": p0.get("compulsory_GBs"),
                              "frac_hbm_compulsory": (p0["compulsory_GBs"] / peaks()[0] if "compulsory_GBs" in p0 else None),
                              "into_store_ms_per_hop": prop[-1]["ms_per_hop"], "nnz": p0["nnz"],
                              "note": "bit-identical to the CPU oracle (tests/test_gpu_propagate*.py); ncu: 64.7 GB of "
                                      "DRAM reads per hop (random 400-B rows miss L2), DESIGN.md §12"}
    except Exception as e:
        out["propagation"] = {"error": repr(e)[:300]}
    try:
        st = _script_lines("bench_storage.py", {"PP_STORAGE_EPOCHS": "1"}, timeout=300)[-1]
        out["storage_tier"] = {k: st.get(k) for k in ("chunk", "storage_mode", "nodes_per_s", "storage_GBs",
                                                      "seq_read_GBs_range", "frac_of_seq_read",
                                                      "frac_of_same_request_seq_read", "sampled_step_bit_exact")}
        out["storage_tier"]["note"] = ("frac_of_seq_read: against the fastest O_DIRECT sequential read of the "
                                       "same files measured before and after the epochs (virtio disk; rate drifts)")
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


def e2e_host_store(pp, torch, cfg, args, W=1, rank=0, local=0, gather_all=None, dist=None, shared_gpu=False):
    """The same epochs end to end from host memory (the paper's host placement):
    the whole store in pinned host memory (N > 1: each rank's shard in a shared memfd spill that
    every peer maps), read zero-copy over PCIe by the gather kernels, so every feature byte crosses
    host -> device inside the timed region; each epoch's node ids are copied back to the host.
    N > 1 uses the weak-scaling shard (products-shaped per rank)."""
    N, H, F, B, chunk = cfg["N"] * W, cfg["H"], cfg["F"], cfg["B"], cfg["chunk"]
    desc = dict(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16,
                hbm_budget_bytes=-1, device=local)
    if W > 1:
        desc.update(world_size=W, rank=rank, peers=pp.PP_PEERS_IPC)
    L = pp.Loader(**desc)
    L.fill_synthetic(DATA_SEED)
    if W > 1:
        pp.pp_import_peer_stores(L.h, b"".join(gather_all(pp.pp_export_store(L.h))))
    stream = torch.cuda.Stream()
    L.set_stream(stream)
    info = L.query()
    steps = info["steps_per_epoch"]
    k = 8
    nslots = min(steps, 2 * k)
    ring = torch.empty((nslots, B, H, F), dtype=torch.bfloat16, device="cuda")
    slots = list(ring.unbind(0))
    nodes = torch.empty((steps, B), dtype=torch.int64, device="cuda")
    host_nodes = torch.empty((steps, B), dtype=torch.int64, pin_memory=True)

    def epoch(e):
        L.epoch_permute(SEED0 + e, chunk, stream)
        done = 0
        while done < steps:
            s0 = done % nslots
            n = min(k, steps - done, nslots - s0)
            done += len(L.next_batches(n, slots[s0], B * H * F * 2, None, nodes[done], stream))
        host_nodes.copy_(nodes, non_blocking=True)

    with torch.cuda.stream(stream):
        epoch(0)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
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
    if dist:
        ms = max(gather_all(ms))
        dist.barrier()
    L.close()
    del ring, slots
    torch.cuda.empty_cache()
    return {"value": N / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": N * info["record_bytes_in"],
            "d2h_bytes_per_step": N * 8, "ms_per_step": ms, "spill_shared": bool(info["spill_shared"]),
            "how": "store in pinned host memory (N > 1: shared memfd spill mapped by every rank), read zero-copy "
                   "over PCIe by the gather kernels, 8 batches per pp_next_batches call; node ids D2H per epoch"}


def cpu_baseline(cfg):
    """SURVEY.md §8(d) oracle timing in both modes: (i) 1 thread, the plain oracle; (ii) all host
    cores (the gather+cast loops under omp parallel for).  Full-N permutation + a bounded sample of
    batches, the epoch extrapolated by rows."""
    nthreads = os.cpu_count() or 1
    out = {}
    for mode, nt, nb in (("one_thread", 1, 8), ("all_cores", nthreads, 32)):
        s, inf = oracle_epoch_sample(cfg, nb, nt)
        out[mode] = {"value": cfg["N"] / s, "threads": nt, "permute_s": inf["permute_s"], "gather_s": inf["gather_s"],
                     "gather_rows": inf["gather_rows"]}
    best = out["all_cores"]
    return {"value": best["value"], "unit": UNIT, "cores": nthreads, "kind": "oracle",
            "sample": (f"full-N permutation (qsort, 1 thread) + gather+cast of {best['gather_rows']} rows "
                       f"({nthreads} OpenMP threads; {out['one_thread']['gather_rows']} rows in the 1-thread mode); "
                       "epoch extrapolated by rows"),
            "modes": out}


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
    ap.add_argument("--skip-nccl", action="store_true", help="N > 1: skip the NCCL all-to-all exchange line")
    ap.add_argument("--skip-papers", action="store_true", help="N > 1: skip the papers100M (configs[2]) line")
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
