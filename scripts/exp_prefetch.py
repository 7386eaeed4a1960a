"""Prefetched-permutation CTA cap sweep: whole products epochs (permute + prefetch + k = 8 gathers)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402

ge.build()
import paper_2504_13266_b200 as pp  # noqa: E402

N, H, F, B = 2_449_029, 4, 100, 8192
steps = -(-N // B)
ring = torch.empty((steps, B, H, F), dtype=torch.bfloat16, device="cuda")
st = torch.cuda.Stream()
for cap in ("0", "32", "64", "148", "296", "0", "64"):
    os.environ["PPLOAD_PREFETCH_CTAS"] = cap
    L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16)
    L.fill_synthetic(2504)
    L.set_stream(st)

    def epoch(e):
        L.epoch_permute(e, 1, st)
        L.epoch_prefetch(e + 1, 1)
        done = 0
        while done < steps:
            done += len(L.next_batches(min(8, steps - done), ring[done], B * H * F * 2, None, None, st))

    with torch.cuda.stream(st):
        for e in range(3):
            epoch(e)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        a.record(st)
        for e in range(20):
            epoch(10 + e)
        b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(json.dumps({"prefetch_ctas": cap, "epoch_ms": ms, "nodes_per_s": N / ms * 1e3}), flush=True)
    L.close()
