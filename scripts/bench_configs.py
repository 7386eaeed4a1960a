"""Secondary single-GPU measurements at the other BASELINE row shapes (one JSON line each).

  products-CR   : configs[1] with chunk reshuffling c = 8192
  papers100M-1r : configs[2] row shape (F = 128, K = 3, fp32 -> bf16, B = 8192, c = 8192) on one
                  rank's store at W = 2 (55.5 M rows, 114 GB, HBM-resident) -- the full 227 GB
                  store does not fit one GPU
  papers100M-labelled : the paper's papers100M setup: a compact store of the
                  1.55 M labelled nodes of 111 M (3.2 GB), RR and c = 8192
  mag240m-1r    : configs[4] row shape (F = 768, K = 3, fp16 -> fp16 copy, B = 8192, RR) on a
                  25 M-row store (154 GB, HBM-resident)
  igb-large-scaled : configs[3] row shape (F = 1024, K = 2, fp32 -> bf16, B = 4096, RR) on a
                  4 M-row store with 13.8 % of the rows in HBM and the rest in pinned host
                  memory read zero-copy (the full 1.2 TB store exceeds this box's 196 GB RAM)
The timed region is whole epochs (permutation prefetched, k = 8 batches per launch) with CUDA events.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402

ge.build()
import paper_2504_13266_b200 as pp  # noqa: E402

PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0


def measure(name, N, H, F, B, chunk, dtype, out_dtype, budget=0, epochs=5, k=8, max_ring_gb=8.0, bound="hbm",
            pcie_peak=None, node_set=None):
    s_in = 4 if dtype == pp.PP_F32 else 2
    s_out = 4 if out_dtype == pp.PP_F32 else 2
    extra = dict(node_set=node_set, store_set_only=True) if node_set is not None else {}
    L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=dtype, batch_size=B, out_dtype=out_dtype,
                  hbm_budget_bytes=budget, **extra)
    N_total = N
    if node_set is not None:
        N = node_set.shape[0]  # positions per epoch
    L.fill_synthetic(2504)
    st = torch.cuda.Stream()
    L.set_stream(st)
    info = L.query()
    steps = info["steps_per_epoch"]
    slot = B * H * F * s_out
    nslots = max(k, min(steps, int(max_ring_gb * 1e9 // slot)))
    ring = torch.empty((nslots, B * H * F * s_out), dtype=torch.uint8, device="cuda")

    def epoch(e):
        L.epoch_permute(e, chunk, st)
        L.epoch_prefetch(e + 1, chunk)
        done = 0
        while done < steps:
            n = min(k, steps - done)
            s0 = done % nslots
            if s0 + n > nslots:
                n = nslots - s0
            done += len(L.next_batches(n, ring[s0], slot, None, None, st))

    with torch.cuda.stream(st):
        epoch(0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        a.record(st)
        for e in range(epochs):
            epoch(1 + e)
        b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / epochs
    per_node = H * F * (s_in + s_out) + 4
    hbm_gbs = N * per_node / ms / 1e6
    out = dict(config=name, N=N, N_total=N_total, H=H, F=F, B=B, chunk=chunk, ms_per_epoch=ms, nodes_per_s=N / ms * 1e3,
               algorithmic_bytes_per_node=per_node, achieved_GBs=hbm_gbs, rows_hbm=info["rows_hbm"],
               rows_spill=info["rows_spill"], ring_slots=nslots)
    if bound == "hbm":
        out.update(bound="hbm", peak=PEAK, frac=hbm_gbs / PEAK)
    else:
        pcie = info["rows_spill"] * H * F * s_in / ms / 1e6
        out.update(bound="pcie", pcie_read_GBs=pcie, peak=pcie_peak, frac=pcie / pcie_peak)
    print(json.dumps(out), flush=True)
    del ring
    L.close()
    torch.cuda.empty_cache()


def dma_peak():
    h = torch.empty(1 << 32, dtype=torch.uint8, pin_memory=True)
    d = torch.empty_like(h, device="cuda")
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    d.copy_(h, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    gbs = h.numel() / a.elapsed_time(b) / 1e6
    del h, d
    torch.cuda.empty_cache()
    return gbs


which = sys.argv[1:] or ["products-CR", "papers100M-1r", "papers100M-labelled", "mag240m-1r", "igb-large-scaled"]
if "products-CR" in which:
    measure("products-CR", 2_449_029, 4, 100, 8192, 8192, pp.PP_F32, pp.PP_BF16, epochs=10)
if "papers100M-1r" in which:
    measure("papers100M-1r", 55_529_978, 4, 128, 8192, 8192, pp.PP_F32, pp.PP_BF16)
if "papers100M-labelled" in which:
    # the paper's own papers100M setup: only the labelled nodes' hop features are
    # kept (0.8 GB per hop, ~1.55 M of 111 M nodes; compact store), so it fits one GPU
    import numpy as np

    S = np.random.default_rng(2504).choice(111_059_956, size=1_546_782, replace=False).astype(np.int64)
    for c in (1, 8192):
        measure(f"papers100M-labelled-c{c}", 111_059_956, 4, 128, 8192, c, pp.PP_F32, pp.PP_BF16, epochs=10,
                node_set=S)
if "mag240m-1r" in which:
    measure("mag240m-1r", 25_000_000, 4, 768, 8192, 1, pp.PP_F16, pp.PP_F16, epochs=3)
if "host-cr" in which:
    # chunk reshuffling over a host-resident store: copy-engine DMA of whole runs (default for
    # c >= 64) vs the zero-copy bulk-copy kernel (PPLOAD_SPILL_PATH=kernel)
    peak = dma_peak()
    print(json.dumps({"pcie_dma_h2d_GBs": peak}), flush=True)
    for path in ("dma", "kernel"):
        os.environ["PPLOAD_SPILL_PATH"] = path
        measure(f"products-host-c8192-{path}", 2_449_029, 4, 100, 8192, 8192, pp.PP_F32, pp.PP_BF16, budget=-1,
                epochs=3, bound="pcie", pcie_peak=peak)
        n = 4_000_000
        measure(f"igb-large-scaled-c4096-{path}", n, 3, 1024, 4096, 4096, pp.PP_F32, pp.PP_BF16,
                budget=int(0.138 * n) * 3 * 1024 * 4, epochs=2, bound="pcie", pcie_peak=peak)
    os.environ.pop("PPLOAD_SPILL_PATH")
if "igb-large-scaled" in which:
    peak = dma_peak()
    print(json.dumps({"pcie_dma_h2d_GBs": peak}), flush=True)
    n = 4_000_000
    measure("igb-large-scaled", n, 3, 1024, 4096, 1, pp.PP_F32, pp.PP_BF16, budget=int(0.138 * n) * 3 * 1024 * 4,
            epochs=2, bound="pcie", pcie_peak=peak)
