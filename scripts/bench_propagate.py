"""§8(f)-2 measurement: pp_propagate (Eq. (2), K = 3 hops) on an ogbn-products-sized synthetic
undirected graph (n = 2,449,029 nodes, 61,859,140 drawn edges -> ~126 M nonzeros of I + A after
symmetrising and dedup, F = 100).  The CSR is built on the GPU with torch (input preparation);
the timed region is pp_propagate only.  One JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402

ge.build()
import paper_2504_13266_b200 as pp  # noqa: E402

n, m, F, K = 2_449_029, 61_859_140, 100, 3
L2FETCH = None
if os.environ.get("PROP_L2FETCH"):  # experiment: the context's max L2 fetch granularity (bytes)
    import ctypes
    torch.zeros(1, device="cuda")
    cu = ctypes.CDLL("libcuda.so.1")
    val = ctypes.c_size_t(int(os.environ["PROP_L2FETCH"]))
    rc = cu.cuCtxSetLimit(ctypes.c_int(5), val)  # CU_LIMIT_MAX_L2_FETCH_GRANULARITY
    got = ctypes.c_size_t(0)
    cu.cuCtxGetLimit(ctypes.byref(got), ctypes.c_int(5))
    L2FETCH = {"set": int(os.environ["PROP_L2FETCH"]), "rc": rc, "got": got.value}
g = torch.Generator(device="cuda").manual_seed(2504)
src = torch.randint(0, n, (m,), device="cuda", generator=g)
dst = torch.randint(0, n, (m,), device="cuda", generator=g)
keep = src != dst
src, dst = src[keep], dst[keep]
diag = torch.arange(n, device="cuda")
keys = torch.cat([src * n + dst, dst * n + src, diag * n + diag])
del src, dst, keep
keys = torch.unique(keys)  # sorted: rows ascending, columns ascending within a row
rows = keys // n
col = (keys % n).contiguous()
del keys
row_ptr = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
row_ptr[1:] = torch.cumsum(torch.bincount(rows, minlength=n), 0)
del rows
nnz = int(row_ptr[-1])
X = torch.randn((n, F), device="cuda", generator=g)
# compulsory DRAM bytes of one hop: X_{k-1} read once, the column ids (int64, as given) and row
# pointers once, X_k written once; the neighbour gathers (nnz rows of F*4 bytes) are L2 traffic when
# the L2-sliced kernel keeps each feature window resident
compulsory = n * F * 4 * 2 + nnz * 8 + (n + 1) * 8
gather_bytes = nnz * F * 4
if os.environ.get("PROP_ONE_HOP"):  # ncu: one hop into the loader store, nothing else
    deg = torch.diff(row_ptr).to(torch.int32)
    L = pp.Loader(data=X, where=pp.PP_MEM_DEVICE, num_nodes=n, num_hops=2, feat_dim=F, hop_stride=0, row_stride=F,
                  dtype=pp.PP_F32, batch_size=8192, out_dtype=pp.PP_BF16)
    L.propagate_store(1, row_ptr, col, deg, torch.cuda.current_stream())
    torch.cuda.synchronize()
    L.close()
    sys.exit(0)
hops = torch.empty((K + 1, n, F), device="cuda")
torch.cuda.synchronize()
pp.pp_propagate(row_ptr, col, X, K, hops)  # warm-up
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 3
a.record()
for _ in range(reps):
    pp.pp_propagate(row_ptr, col, X, K, hops)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
# algorithmic bytes: per hop every nonzero reads its neighbour row (F*4) + column (8) + weight (8),
# every row writes F*4 and reads 2 row pointers; plus the weights pass and the hop-0 copy
per_hop = nnz * (F * 4 + 16) + n * (F * 4 + 16)
total = K * per_hop + nnz * (8 + 8 + 16) + 2 * n * F * 4
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
print(json.dumps({"config": "products-sized ER graph", "n": n, "nnz": nnz, "F": F, "K": K, "ms": ms,
                  "algorithmic_GBs": total / ms / 1e6, "frac_hbm": total / ms / 1e6 / peak,
                  "ms_per_hop": ms / K, "compulsory_bytes_per_hop": compulsory,
                  "compulsory_GBs": compulsory * K / ms / 1e6, "gather_bytes_per_hop": gather_bytes,
                  "gather_GBs": gather_bytes * K / ms / 1e6,
                  "kernel": os.environ.get("PPLOAD_SPMM", "auto (row kernels; PPLOAD_SPMM=sliced opt-in)"),
                  "l2_fetch": L2FETCH}))

# Same graph, propagated INTO a loader store (pp_propagate_store: node-major [n, K+1, F] fp32
# records, hop slot k from slot k-1, weights from the degree array on the fly).
del hops
deg = torch.diff(row_ptr).to(torch.int32)
L = pp.Loader(data=X, where=pp.PP_MEM_DEVICE, num_nodes=n, num_hops=K + 1, feat_dim=F, hop_stride=0, row_stride=F,
              dtype=pp.PP_F32, batch_size=8192, out_dtype=pp.PP_BF16)
s = torch.cuda.current_stream()


def store_pass():
    for k in range(1, K + 1):
        L.propagate_store(k, row_ptr, col, deg, s)


store_pass()
torch.cuda.synchronize()
a.record()
for _ in range(reps):
    store_pass()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
per_hop = nnz * (F * 4 + 8 + 4) + n * (F * 4 + 16)
print(json.dumps({"config": "products-sized ER graph, into the loader store",
                  "kernel": os.environ.get("PPLOAD_SPMM", "auto (row kernels; PPLOAD_SPMM=sliced opt-in)"), "n": n,
                  "nnz": nnz, "F": F, "K": K, "ms": ms, "algorithmic_GBs": K * per_hop / ms / 1e6,
                  "compulsory_GBs": compulsory * K / ms / 1e6, "gather_GBs": gather_bytes * K / ms / 1e6,
                  "frac_hbm": K * per_hop / ms / 1e6 / peak, "ms_per_hop": ms / K, "l2_fetch": L2FETCH}))
L.close()
