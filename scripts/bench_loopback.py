"""§8(e) sharded path on one GPU: products-shaped store (N = 2,449,029, F = 100, K = 3) split
round-robin over W loopback shards (PP_PEERS_LOOPBACK: W loader handles in one process, the
"peer" stores are local HBM allocations), every rank assembling its slice of every step of
the global epoch with the sharded gather kernel (owner table, exchange-copy reads of remote
rows).  No NVLink is involved: this measures the sharded kernel's own efficiency, not the
link.  Timed: whole epochs of all W ranks (k = 8 steps per launch), CUDA events.  One JSON
line per W.  LOOPBACK_EXCHANGE=a2a: the all-to-all path instead (count table at the permute;
per step the index kernel, the pack by the gather kernel straight into the receive buffer and the
unpack -- the NCCL transfer itself is what loopback skips)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402

ge.build()
import paper_2504_13266_b200 as pp  # noqa: E402

N, H, F, B, K = 2_449_029, 4, 100, 8192, 8
PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
st = torch.cuda.Stream()
A2A = os.environ.get("LOOPBACK_EXCHANGE") == "a2a"
if A2A:
    os.environ["PPLOAD_EXCHANGE"] = "a2a"
for W in ((2, 4, 8) if A2A else (1, 2, 4, 8)):
    Ls = []
    for r in range(W):
        kw = dict(world_size=W, rank=r, peers=pp.PP_PEERS_LOOPBACK) if W > 1 else {}
        L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16, **kw)
        L.fill_synthetic(2504)
        Ls.append(L)
    if W > 1:
        pp.pp_link_loopback([L.h for L in Ls])
    for L in Ls:
        L.set_stream(st)
    steps = Ls[0].query()["steps_per_epoch"]
    xcast = Ls[0].query()["exchange_cast"]
    ring = torch.empty((steps * W, B, H, F), dtype=torch.bfloat16, device="cuda")  # one slot per (rank, step)
    slot = B * H * F * 2

    def epoch(e, evs=None):
        for L in Ls:  # every rank computes the same global order (on W GPUs these run in parallel)
            L.epoch_permute(e, 1, st)
        if evs:
            evs[0].record(st)
        for r, L in enumerate(Ls):
            done = 0
            while done < steps:
                done += len(L.next_batches(min(K, steps - done), ring[r * steps + done], slot, None, None, st))
        if evs:
            evs[1].record(st)

    with torch.cuda.stream(st):
        epoch(0)
    torch.cuda.synchronize()
    reps = 5
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    with torch.cuda.stream(st):
        for e in range(reps):
            epoch(1 + e, evs[e])
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in evs) / reps  # the gathers of all ranks (permutations excluded)
    # HBM bytes per node: local rows fp32 (1600), remote rows from the exchange copy (800) or fp32
    remote = (W - 1) / W
    rd = (1 - remote) * H * F * 4 + remote * H * F * (2 if xcast else 4)
    per_node = rd + H * F * 2 + 4
    if A2A:  # pack: fp32 record read + cast row written; unpack: cast row read + written; + order
        per_node = H * F * 4 + 3 * H * F * 2 + 4
    print(json.dumps({"W": W, "exchange": "a2a (loopback, no transport)" if A2A else "peer reads",
                      "exchange_cast": bool(xcast), "gather_ms_per_epoch_all_ranks": ms, "nodes_per_s": N / ms * 1e3,
                      "hbm_bytes_per_node": per_node, "achieved_GBs": N * per_node / ms / 1e6,
                      "frac_hbm": N * per_node / ms / 1e6 / PEAK,
                      "note": "gathers of all W ranks, serialised on one GPU; permutations excluded"}),
          flush=True)
    del ring
    for L in Ls:
        L.close()
    torch.cuda.empty_cache()
