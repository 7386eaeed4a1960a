"""§8(f)-1 measurement: fused gather + per-hop linear (tcgen05) vs the unfused pipeline
(loader gather into a bf16 batch, then torch.bmm / cuBLAS per hop) on the products shape
with SIGN's hidden size 512.  One JSON line per variant; whole epochs
(permutation prefetched) timed with CUDA events."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402

ge.build()
import paper_2504_13266_b200 as pp  # noqa: E402

N, H, F, B, D = 2_449_029, 4, 100, 8192, 512
K = int(os.environ.get("LIN_K", "8"))  # steps per launch
PEAK_HBM = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
PEAK_TF = json.load(open("MEASURED_PEAKS.json"))["bf16_tflops"] if os.path.exists("MEASURED_PEAKS.json") else 1590.0
L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16)
L.fill_synthetic(2504)
st = torch.cuda.Stream()
L.set_stream(st)
steps = L.query()["steps_per_epoch"]
rng = np.random.default_rng(0)
W = torch.from_numpy((rng.standard_normal((H, F, D)) / 10).astype(np.float32)).cuda().to(torch.bfloat16)
nslots = steps  # one Z slot per step of the epoch (10 GB): no slot is rewritten while an overlapped launch may still write it
Z = torch.empty((nslots, B, H, D), dtype=torch.bfloat16, device="cuda")
X = torch.empty((nslots, B, H, F), dtype=torch.bfloat16, device="cuda")
Zh = torch.empty((nslots, H, B, D), dtype=torch.bfloat16, device="cuda")  # unfused output, hop-major
zs = B * H * D * 2
xs = B * H * F * 2


def fused_epoch(e):
    L.epoch_permute(e, 1, st)
    L.epoch_prefetch(e + 1, 1)
    done = 0
    while done < steps:
        s0 = done % nslots
        n = min(K, steps - done, nslots - s0)
        done += len(L.next_batches_linear(n, W, D, Z[s0], "bf16", zs, st))


def unfused_epoch(e):
    L.epoch_permute(e, 1, st)
    L.epoch_prefetch(e + 1, 1)
    done = 0
    while done < steps:
        s0 = done % nslots
        n = min(K, steps - done, nslots - s0)
        got = L.next_batches(n, X[s0], xs, None, None, st)
        for i in range(len(got)):  # per hop: [B, F] @ [F, D] on cuBLAS (torch.bmm over hops)
            torch.bmm(X[s0 + i].transpose(0, 1), W, out=Zh[s0 + i])
        done += len(got)


def timeit(fn, reps=5):
    with torch.cuda.stream(st):
        fn(0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        a.record(st)
        for r in range(reps):
            fn(1 + r)
        b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


# variants timed in interleaved rounds (box-to-box and power-state drift hits all alike); the
# fused kernel is the K-chunked one by default (round 2), PPLOAD_LINEAR=res selects the W-resident one
VARIANTS = [("fused_tcgen05", fused_epoch, "", H * F * 4 + H * D * 2 + 4),
            ("fused_tcgen05_resident", fused_epoch, "res", H * F * 4 + H * D * 2 + 4),
            ("unfused_gather_then_cublas", unfused_epoch, "", H * F * 4 + H * F * 2 + 4 + H * F * 2 + H * D * 2)]
times = {v[0]: [] for v in VARIANTS}
for rnd in range(int(os.environ.get("LIN_ROUNDS", "3"))):
    for name, fn, mode, _ in VARIANTS:
        os.environ["PPLOAD_LINEAR"] = mode
        times[name].append(timeit(fn))
os.environ.pop("PPLOAD_LINEAR", None)
for name, fn, mode, bytes_per_row in VARIANTS:
    ms = float(np.median(times[name]))
    flops = 2.0 * N * H * F * D
    print(json.dumps({"variant": name, "steps_per_launch": K, "ms_per_epoch": ms, "rounds_ms": times[name],
                      "nodes_per_s": N / ms * 1e3,
                      "hbm_bytes_per_row": bytes_per_row, "achieved_GBs": N * bytes_per_row / ms / 1e6,
                      "frac_hbm": N * bytes_per_row / ms / 1e6 / PEAK_HBM,
                      "tflops": flops / ms / 1e9, "frac_tensor": flops / ms / 1e9 / PEAK_TF}), flush=True)
L.close()

if "--debug" in sys.argv:  # which stage bounds the fused kernel (bits: see LinearArgs::debug)
    i = sys.argv.index("--debug")
    dbgs = sys.argv[i + 1].split(",") if i + 1 < len(sys.argv) else ["1", "2", "3"]
    for dbg in dbgs:
        os.environ["PPLOAD_DEBUG_LINEAR"] = dbg
        L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16)
        L.fill_synthetic(2504)
        L.set_stream(st)
        print(json.dumps({"variant": f"fused_debug{dbg}", "ms_per_epoch": timeit(fused_epoch)}), flush=True)
        L.close()
    os.environ.pop("PPLOAD_DEBUG_LINEAR")
