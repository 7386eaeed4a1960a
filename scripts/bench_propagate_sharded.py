"""§8(f)-2 sharded propagation on one GPU: the products-sized Erdős–Rényi graph of
bench_propagate.py propagated into loader stores split over W loopback shards
(pp_propagate_store: every shard computes hop slot k of its own rows from hop slot k-1 of all
owners; the "peer" stores are local HBM, so this measures the sharded kernel, not NVLink).
Time: K = 3 hops of all W shards, serialised on one GPU.  One JSON line per W."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402

ge.build()
import paper_2504_13266_b200 as pp  # noqa: E402

n, m, F, K = 2_449_029, 61_859_140, 100, 3
PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
g = torch.Generator(device="cuda").manual_seed(2504)
src = torch.randint(0, n, (m,), device="cuda", generator=g)
dst = torch.randint(0, n, (m,), device="cuda", generator=g)
keep = src != dst
src, dst = src[keep], dst[keep]
diag = torch.arange(n, device="cuda")
keys = torch.unique(torch.cat([src * n + dst, dst * n + src, diag * n + diag]))
del src, dst, keep
rows = keys // n
col = (keys % n).contiguous()
del keys
counts = torch.bincount(rows, minlength=n)
row_ptr = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
row_ptr[1:] = torch.cumsum(counts, 0)
deg = counts.to(torch.int32)
nnz = int(row_ptr[-1])
X = torch.randn((n, F), device="cuda", generator=g)
st = torch.cuda.current_stream()

for W in (1, 2, 4):
    Ls, csrs = [], []
    for r in range(W):
        kw = dict(world_size=W, rank=r, peers=pp.PP_PEERS_LOOPBACK) if W > 1 else {}
        Ls.append(pp.Loader(data=X, where=pp.PP_MEM_DEVICE, num_nodes=n, num_hops=K + 1, feat_dim=F, hop_stride=0,
                            row_stride=F, dtype=pp.PP_F32, batch_size=8192, out_dtype=pp.PP_BF16, **kw))
        mine = torch.arange(r, n, W, device="cuda")  # this shard's rows, local order
        lens = counts[mine]
        lrp = torch.zeros(mine.numel() + 1, dtype=torch.int64, device="cuda")
        lrp[1:] = torch.cumsum(lens, 0)
        idx = torch.repeat_interleave(row_ptr[mine], lens) + (torch.arange(int(lrp[-1]), device="cuda") -
                                                               torch.repeat_interleave(lrp[:-1], lens))
        csrs.append((lrp, col[idx].contiguous()))
        del mine, lens, idx
    if W > 1:
        pp.pp_link_loopback([L.h for L in Ls])

    def run():
        for k in range(1, K + 1):
            for L, (lrp, lci) in zip(Ls, csrs):
                L.propagate_store(k, lrp, lci, deg, st)

    run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 2
    a.record(st)
    for _ in range(reps):
        run()
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    per_hop = nnz * (F * 4 + 8 + 4) + n * (F * 4 + 16)
    print(json.dumps({"W": W, "nnz": nnz, "ms_per_hop_all_shards": ms / K, "algorithmic_GBs": K * per_hop / ms / 1e6,
                      "frac_hbm": K * per_hop / ms / 1e6 / PEAK,
                      "note": "loopback shards on one GPU (peer rows are local HBM); bit-exactness: "
                              "tests/test_gpu_propagate_store.py"}), flush=True)
    for L in Ls:
        L.close()
    del Ls, csrs
    torch.cuda.empty_cache()
