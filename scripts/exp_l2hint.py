"""L2 prefetch-hint sweep for the products gather (k = 8 per launch, no permutation overlap)."""
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
for hint in ("0", "1", "2", "0", "2"):
    for tile in ("16", "32"):
        os.environ["PPLOAD_L2_PREFETCH"] = hint
        os.environ["PPLOAD_TILE_ROWS"] = tile
        L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16)
        L.fill_synthetic(2504)
        L.set_stream(st)
        L.epoch_permute(1, 1, st)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        times = []
        for rep in range(12):
            L.seek(0)
            ev[0].record(st)
            done = 0
            while done < steps:
                done += len(L.next_batches(min(8, steps - done), ring[done], B * H * F * 2, None, None, st))
            ev[1].record(st)
            torch.cuda.synchronize()
            if rep >= 2:
                times.append(ev[0].elapsed_time(ev[1]))
        ms = sorted(times)[len(times) // 2]
        print(json.dumps({"l2_hint": hint, "tile": tile, "gather_ms": ms, "GBs": N * 2404 / ms / 1e6}), flush=True)
        L.close()
