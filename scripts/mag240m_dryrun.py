"""BASELINE configs[4] (MAG240M-shaped: 244,160,499 nodes, F = 768, K = 3, fp16, W = 8, round-robin)
as rank 7 of 8 on ONE GPU: pp_loader_create of the full per-rank shard (30.5 M records of 6144 B,
187.5 GB) with the automatic HBM budget; rows that do not fit go to the shared host spill (memfd,
PP_PEERS_IPC).  Prints the memory plan, fills the shard with the §8(d) generator G16, checks sampled
records against the oracle, and times locality-aware epochs (pp_epoch_permute_local: this rank's
own rows, HBM + spill; no peers are needed) with sampled batches checked element-wise.
One JSON line per measurement on stdout."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402

ge.build()
import oracle  # noqa: E402
import paper_2504_13266_b200 as pp  # noqa: E402

N, H, F, B, W, RANK = 244_160_499, 4, 768, 8192, 8, 7
N = int(os.environ.get("MAG_N", N))
free0, total = torch.cuda.mem_get_info()
t0 = time.time()
L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F16, batch_size=B, out_dtype=pp.PP_F16,
              world_size=W, rank=RANK, peers=pp.PP_PEERS_IPC)
t_create = time.time() - t0
q = L.query()
free1, _ = torch.cuda.mem_get_info()
plan = {k: q[k] for k in ("local_rows", "rows_hbm", "rows_spill", "record_bytes_in", "spill_shared", "hbm_store_bytes",
                          "hbm_exchange_bytes", "hbm_scratch_bytes", "host_spill_bytes")}
print(json.dumps({"what": "mag240m_rank7_memory_plan", "num_nodes": N, "world_size": W, "rank": RANK,
                  "gpu_total_bytes": total, "gpu_free_before": free0, "gpu_free_after_create": free1,
                  "create_s": t_create, **plan,
                  "hbm_fraction_of_shard": q["rows_hbm"] / q["local_rows"]}), flush=True)
t0 = time.time()
L.fill_synthetic(2504)
t_fill = time.time() - t0
rng = np.random.default_rng(1)
lr = np.concatenate([rng.integers(0, q["local_rows"], 6), [0, q["rows_hbm"] - 1, q["local_rows"] - 1]])
if q["rows_spill"] > 0:
    lr = np.concatenate([lr, [q["rows_hbm"], q["rows_hbm"] + q["rows_spill"] // 2]])
lr = np.unique(lr)
ok = True
for r in lr:
    got = L.read_store(int(r), 1)[0].view(np.uint16).reshape(H, F)
    want = oracle.gen_rows(2504, oracle.F16, H, F, np.array([int(r) * W + RANK]))[0]
    ok &= bool(np.array_equal(got, want))
print(json.dumps({"what": "mag240m_rank7_fill", "fill_s": t_fill, "sampled_records_match_oracle": ok,
                  "sampled_local_rows": lr.tolist()}), flush=True)

st = torch.cuda.Stream()
L.set_stream(st)
steps = -(-q["local_rows"] // B)
k = 8
ring = torch.empty((k, B, H, F), dtype=torch.float16, device="cuda")
nodes = torch.empty((k, B), dtype=torch.int64, device="cuda")
slot = B * H * F * 2


def epoch(seed, check=False):
    L.epoch_permute_local(seed, 1, st)
    done, bad = 0, 0
    checks = {0, steps // 2, steps - 1}
    while done < steps:
        rows = L.next_batches(min(k, steps - done), ring, slot, None, nodes if check else None, st)
        if check and any(done + i in checks for i in range(len(rows))):
            st.synchronize()
            for i, nr in enumerate(rows):
                if done + i in checks:
                    v = nodes[i, :nr].cpu().numpy()
                    want = oracle.gen_rows(2504, oracle.F16, H, F, v[:512])
                    got = ring[i, :min(nr, 512)].view(torch.int16).cpu().numpy().view(np.uint16)
                    bad += int(not np.array_equal(got, want)) + int(not np.all(v % W == RANK))
        done += len(rows)
    return bad


with torch.cuda.stream(st):
    bad = epoch(250413266, check=True)
    st.synchronize()
    # local order must be the oracle's local epoch mapped to global ids (sampled)
    order = L.get_order()
    want = oracle.epoch_order(250413266, q["local_rows"], 1) * W + RANK if q["local_rows"] < 40_000_000 else None
    order_ok = bool(np.array_equal(order, want)) if want is not None else None
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    reps = 2
    for e in range(reps):
        epoch(250413267 + e)
    b.record(st)
    st.synchronize()
ms = a.elapsed_time(b) / reps
rows_hbm, rows_spill = q["rows_hbm"], q["rows_spill"]
rec = q["record_bytes_in"]
print(json.dumps({"what": "mag240m_rank7_local_epoch", "ms_per_epoch": ms, "nodes_per_s": q["local_rows"] / (ms / 1e3),
                  "bytes_per_node": 2 * rec + 4, "achieved_GBs": q["local_rows"] * (2 * rec + 4) / ms / 1e6,
                  "pcie_GBs_spilled_rows": rows_spill * rec / ms / 1e6, "batches_bad": bad, "local_order_ok": order_ok,
                  "note": "pp_epoch_permute_local over this rank's 30.5 M rows: HBM rows + shared-spill rows (PCIe)"}),
      flush=True)
L.close()
