"""§8(f)-1 at the wide BASELINE row shapes: the K-chunked fused gather + per-hop linear
(k_gather_linear_kc) on IGB-large rows (F = 1024, K = 2, fp32 store -> bf16, B = 4096) and MAG240M
rows (F = 768, K = 3, fp16 store, B = 8192), SIGN's hidden 512, bf16 Z.  Stores of
LIN_ROWS records (default 4 M: 49 / 25 GB), HBM-resident, SGD-RR epochs with the next order prefetched,
8 steps per launch.  Reports nodes/s, HBM GB/s by algorithmic bytes (H F s_in read + H D 2 written
+ 4 per node) and tensor TFLOP/s (2 H F D per node) against MEASURED_PEAKS.json.  One JSON line per
shape."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402

ge.build()
import paper_2504_13266_b200 as pp  # noqa: E402

ROWS = int(os.environ.get("LIN_ROWS", 4_000_000))
K = int(os.environ.get("LIN_K", "8"))
D = 512
pk = json.load(open("MEASURED_PEAKS.json")) if os.path.exists("MEASURED_PEAKS.json") else {}
PEAK_HBM = pk.get("hbm_gbs", 6650.0)
PEAK_TF = pk.get("bf16_tflops", 1590.0)
PEAK_TF_SUST = pk.get("bf16_tflops_sustained", PEAK_TF)  # back-to-back cuBLAS for seconds (power-capped clocks)
SHAPES = {"products": dict(H=4, F=100, B=8192, dtype=pp.PP_F32, out=pp.PP_BF16, s_in=4, rows=2_449_029),
          "igb_large": dict(H=3, F=1024, B=4096, dtype=pp.PP_F32, out=pp.PP_BF16, s_in=4),
          "mag240m": dict(H=4, F=768, B=8192, dtype=pp.PP_F16, out=pp.PP_F16, s_in=2)}
for name in os.environ.get("LIN_SHAPES", "igb_large,mag240m").split(","):
    c = SHAPES[name]
    H, F, B = c["H"], c["F"], c["B"]
    ROWS = c.get("rows", int(os.environ.get("LIN_ROWS", 4_000_000)))
    L = pp.Loader(num_nodes=ROWS, num_hops=H, feat_dim=F, dtype=c["dtype"], batch_size=B, out_dtype=c["out"])
    L.fill_synthetic(2504)
    st = torch.cuda.Stream()
    L.set_stream(st)
    steps = L.query()["steps_per_epoch"]
    wdt = torch.bfloat16 if c["out"] == pp.PP_BF16 else torch.float16
    W = (torch.randn((H, F, D), device="cuda") / np.sqrt(F)).to(wdt)
    zs = B * H * D * 2
    nslots = min(steps, max(K, int(16e9 // zs)))
    Z = torch.empty((nslots, B, H, D), dtype=torch.bfloat16, device="cuda")

    def epoch(e):
        L.epoch_permute(e, 1, st)
        L.epoch_prefetch(e + 1, 1)
        done = 0
        while done < steps:
            s0 = done % nslots
            n = min(K, steps - done, nslots - s0)
            done += len(L.next_batches_linear(n, W, D, Z[s0], "bf16", zs, st))

    with torch.cuda.stream(st):
        epoch(0)
    torch.cuda.synchronize()

    def timed(reps=3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a.record(st)
            for r in range(reps):
                epoch(1 + r)
            b.record(st)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    # LIN_AB="d1,d2": interleaved A/B of PPLOAD_DEBUG_LINEAR values in this process (box-to-box clock
    # and power differences would swamp a few per cent between separate runs)
    ab = os.environ.get("LIN_AB")
    if ab:
        vals = ab.split(",")
        res = {v: [] for v in vals}
        for rnd in range(4):
            for v in vals:
                # a token is a PPLOAD_DEBUG_LINEAR value, or "E:NAME=VAL+NAME2=VAL2" (environment settings)
                saved = {}
                if v.startswith("E:"):
                    os.environ["PPLOAD_DEBUG_LINEAR"] = "0"
                    for kv in v[2:].split("+"):
                        key, val = kv.split("=", 1)
                        saved[key] = os.environ.get(key)
                        os.environ[key] = val
                else:
                    os.environ["PPLOAD_DEBUG_LINEAR"] = v
                res[v].append(timed(2))
                for key, old in saved.items():
                    if old is None:
                        os.environ.pop(key, None)
                    else:
                        os.environ[key] = old
        os.environ.pop("PPLOAD_DEBUG_LINEAR")
        print(json.dumps({"shape": name, "ab_ms_per_epoch": {v: sorted(x) for v, x in res.items()},
                          "ab_median_ms": {v: sorted(x)[len(x) // 2] for v, x in res.items()}}), flush=True)
    import bench  # the NVML clock sampler of the bench line

    clk = bench.ClockSampler(torch.cuda.current_device())
    with clk:
        ms = timed()
    clocks = clk.summary()
    per_node = H * F * c["s_in"] + H * D * 2 + 4
    flops = 2.0 * H * F * D
    print(json.dumps({"shape": name, "debug": os.environ.get("PPLOAD_DEBUG_LINEAR", "0"), "rows": ROWS, "H": H, "F": F, "B": B, "D": D, "steps_per_launch": K,
                      "ms_per_epoch": ms, "nodes_per_s": ROWS / ms * 1e3, "hbm_bytes_per_node": per_node,
                      "achieved_GBs": ROWS * per_node / ms / 1e6, "frac_hbm": ROWS * per_node / ms / 1e6 / PEAK_HBM,
                      "tflops": ROWS * flops / ms / 1e9, "frac_tensor": ROWS * flops / ms / 1e9 / PEAK_TF,
                      "frac_tensor_sustained": ROWS * flops / ms / 1e9 / PEAK_TF_SUST,
                      "w_l2_bytes_per_node": H * F * D * 2 / 128, "clocks": clocks}), flush=True)
    L.close()
    del Z
    torch.cuda.empty_cache()
