"""Gather efficiency vs record size and batch size (SGD-RR, fp32 store -> bf16 batches, H = 4,
HBM-resident, k = 8 batches per launch, next order prefetched).  The store is ~4 GB for every F
(N = 4 GB / record), so it never fits L2; outputs rotate over >= 1 GB.  One JSON line per point:
whole-epoch nodes/s and algorithmic GB/s against the measured HBM copy peak."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402

ge.build()
import paper_2504_13266_b200 as pp  # noqa: E402

PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
H, K = 4, 8
st = torch.cuda.Stream()


def point(F, B, epochs=5):
    rec = H * F * 4
    N = int(4e9 // rec)
    L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16)
    L.fill_synthetic(2504)
    L.set_stream(st)
    steps = L.query()["steps_per_epoch"]
    slot = B * H * F * 2
    nslots = min(steps, max(K, int(2e9 // slot)))
    ring = torch.empty((nslots, slot), dtype=torch.uint8, device="cuda")
    slots = list(ring.unbind(0))

    def epoch(e):
        L.epoch_permute(e, 1, st)
        L.epoch_prefetch(e + 1, 1)
        done = 0
        while done < steps:
            s0 = done % nslots
            n = min(K, steps - done, nslots - s0)
            done += len(L.next_batches(n, slots[s0], slot, None, None, st))

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
    per_node = H * F * 6 + 4
    gbs = N * per_node / ms / 1e6
    print(json.dumps({"F": F, "record_bytes": rec, "B": B, "N": N, "ms_per_epoch": ms, "nodes_per_s": N / ms * 1e3,
                      "achieved_GBs": gbs, "frac_hbm": gbs / PEAK}), flush=True)
    del ring, slots
    L.close()
    torch.cuda.empty_cache()


for F in (8, 16, 32, 64, 100, 128, 256, 512, 1024):
    point(F, 8192)
for B in (1024, 2048, 4096, 16384, 65536):
    point(100, B)
