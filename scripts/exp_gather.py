"""Launch-configuration sweep for the products gather (tile rows x PDL x batches per call).
Prints one JSON line per configuration; used to pick the library defaults."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402

ge.build()
import paper_2504_13266_b200 as pp  # noqa: E402

N, H, F, B = 2_449_029, 4, 100, 8192
steps = -(-N // B)
ring = torch.empty((steps, B, H, F), dtype=torch.bfloat16, device="cuda")
slot = B * H * F * 2
stream = torch.cuda.Stream()


def run(tile, pdl, gps, k, prefetch, chunk=1, reps=10):
    os.environ["PPLOAD_TILE_ROWS"] = str(tile)
    os.environ["PPLOAD_PDL"] = str(pdl)
    os.environ["PPLOAD_GRID_PER_SM"] = str(gps)
    L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16)
    L.fill_synthetic(2504)
    L.set_stream(stream)
    host = []

    def epoch(e, ev=None):
        L.epoch_permute(e, chunk, stream)
        if prefetch:
            L.epoch_prefetch(e + 1, chunk)
        if ev is not None:
            ev.record(stream)
        t0 = time.perf_counter()
        done = 0
        while done < steps:
            if k == 1:
                L.next_batch(ring[done], None, None, stream)
                done += 1
            else:
                done += len(L.next_batches(min(k, steps - done), ring[done], slot, None, None, stream))
        host.append(time.perf_counter() - t0)

    with torch.cuda.stream(stream):
        for e in range(3):
            epoch(e)
    torch.cuda.synchronize()
    host.clear()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(reps)]
    with torch.cuda.stream(stream):
        for i in range(reps):
            evs[i][0].record(stream)
            epoch(100 + i, evs[i][1])
            evs[i][2].record(stream)
    torch.cuda.synchronize()
    ep = sorted(a.elapsed_time(c) for a, b, c in evs)[reps // 2]
    ga = sorted(b.elapsed_time(c) for a, b, c in evs)[reps // 2]
    L.close()
    bytes_epoch = N * (1600 + 800 + 4)
    print(json.dumps(dict(tile=tile, pdl=pdl, gps=gps, k=k, prefetch=prefetch, chunk=chunk, epoch_ms=ep, gather_ms=ga,
                          nodes_per_s=N / ep * 1e3, gather_GBs=bytes_epoch / ga / 1e6,
                          host_us_per_call=1e6 * sorted(host)[len(host) // 2] / (steps if k == 1 else -(-steps // k)))),
          flush=True)


for tile in (8, 16, 32):
    for pdl in (0, 1):
        run(tile, pdl, 4, 1, 0)
for k in (2, 4, 8, 16, 299):
    run(16, 1, 4, k, 0)
for gps in (2, 8):
    run(16, 1, gps, 299, 0)
run(16, 1, 4, 1, 1)
run(16, 1, 4, 8, 1)
run(16, 1, 4, 299, 1)
run(16, 1, 4, 8, 1, chunk=8192)
run(16, 1, 4, 299, 1, chunk=8192)

# --- bulk-copy (TMA) path vs register-staged LDG path, HBM and pinned-host stores
def run_store(mode, budget, k, reps=3, chunk=1):
    os.environ["PPLOAD_GATHER"] = mode
    os.environ["PPLOAD_TILE_ROWS"] = "16"
    L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16,
                  hbm_budget_bytes=budget)
    L.fill_synthetic(2504)
    L.set_stream(stream)

    def epoch(e):
        L.epoch_permute(e, chunk, stream)
        done = 0
        while done < steps:
            done += len(L.next_batches(min(k, steps - done), ring[done], slot, None, None, stream))

    with torch.cuda.stream(stream):
        epoch(0)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        a.record(stream)
        for i in range(reps):
            epoch(1 + i)
        b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    info = L.query()
    L.close()
    print(json.dumps(dict(mode=mode, budget=budget, k=k, chunk=chunk, epoch_ms=ms, nodes_per_s=N / ms * 1e3,
                          rows_spill=info["rows_spill"], read_GBs=N * 1600 / ms / 1e6)), flush=True)


for mode in ("ldg", "tma"):
    run_store(mode, 0, 8, reps=10)
    run_store(mode, 0, 299, reps=10)
    run_store(mode, -1, 8)
    run_store(mode, -1, 8, chunk=8192)
# DMA reference: one 3.9 GB pinned host -> device copy
h = torch.empty(N * 1600, dtype=torch.uint8, pin_memory=True)
d = torch.empty_like(h, device="cuda")
d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True)
b = torch.cuda.Event(enable_timing=True)
a.record()
d.copy_(h, non_blocking=True)
b.record()
torch.cuda.synchronize()
print(json.dumps(dict(dma_h2d_GBs=h.numel() / a.elapsed_time(b) / 1e6)), flush=True)
