"""§8(a) A6 measurement: the paper's double-buffer prefetch (1.33x average with
GPU-resident hop features on its RTX A6000 server) on one B200.

Consumer: a SIGN-style training step on each batch, written with plain torch ops (cuBLAS) --
per-hop linear (F -> 512) for every hop, concat, Linear(4*512 -> 512), ReLU, Linear(512 -> 47),
cross-entropy, backward, SGD update (hidden 512; 47 classes as ogbn-products).
It only exists to give the loader something to overlap with; nothing here is a model or
training framework.

  serial : pp_next_batch and the step on ONE stream (the loader's work is on the critical path)
  double : the loader on its own stream filling two buffers alternately, the step on the
           consumer stream; per-buffer events (pp_next_batches_ev) order them (the paper's design)
  double_<n>ctas: the same with the gather grid capped at n CTAs (pp_set_grid_limit), so the
           consumer keeps most SMs while batches are assembled
  compute: the step alone on a resident batch (lower bound)
One JSON line per mode; products-shaped store (N = 2,449,029, F = 100, K = 3), B = 8192, RR;
DB_PLACEMENT=hbm (default) or host (the store in pinned host memory, read over PCIe)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402

ge.build()
import paper_2504_13266_b200 as pp  # noqa: E402

N, H, F, B, D, C = 2_449_029, 4, 100, 8192, 512, 47
EPOCHS = int(os.environ.get("DB_EPOCHS", "3"))
torch.manual_seed(0)
dev = "cuda"
W1 = (torch.randn(H, F, D, device=dev) / 10).to(torch.bfloat16).requires_grad_()
W2 = (torch.randn(H * D, D, device=dev) / 40).to(torch.bfloat16).requires_grad_()
W3 = (torch.randn(D, C, device=dev) / 20).to(torch.bfloat16).requires_grad_()
params = [W1, W2, W3]
labels_all = torch.randint(0, C, (N,), dtype=torch.int64)


GRAPH = os.environ.get("DB_GRAPH", "0") == "1"  # capture the consumer step in CUDA graphs (GPU-bound step)
graphs = {}


def step(x, y):
    if GRAPH and x.shape[0] == B and (x.data_ptr(), y.data_ptr()) in graphs:
        graphs[(x.data_ptr(), y.data_ptr())].replay()
        return
    _step(x, y)


def _step(x, y):
    # x: [rows, H, F] bf16 batch, y: [rows] labels
    z = torch.bmm(x.transpose(0, 1), W1)             # [H, rows, D] per-hop linear
    h = torch.relu(z.transpose(0, 1).reshape(x.shape[0], H * D))
    h = torch.relu(h @ W2)
    loss = torch.nn.functional.cross_entropy((h @ W3).float(), y)
    loss.backward()
    with torch.no_grad():
        for p in params:
            p -= 1e-3 * p.grad
            p.grad = None


CHUNK = int(os.environ.get("DB_CHUNK", "1"))  # 1: SGD-RR; c > 1: chunk reshuffling (host rows then move by DMA)
PLACEMENT = os.environ.get("DB_PLACEMENT", "hbm")  # hbm: GPU-resident store; host: pinned host memory (UVA)
L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16,
              labels=labels_all.numpy().astype("int32"), hbm_budget_bytes=-1 if PLACEMENT == "host" else 0)
L.fill_synthetic(2504)
steps = L.query()["steps_per_epoch"]
bufs = [torch.empty((B, H, F), dtype=torch.bfloat16, device=dev) for _ in range(2)]
labs = [torch.zeros(B, dtype=torch.int32, device=dev) for _ in range(2)]
cons = torch.cuda.Stream()
_prio = {"high": -5, "low": 0, "normal": 0}[os.environ.get("DB_LOADER_PRIO", "normal")]  # torch clamps to range
loader_stream = torch.cuda.Stream(priority=_prio) if os.environ.get("DB_LOADER_PRIO") == "high" else torch.cuda.Stream()
if GRAPH:  # one graph per (batch buffer, label buffer) pair; the ragged last batch runs eagerly
    ylong = [torch.zeros(B, dtype=torch.int64, device=dev) for _ in range(2)]
    with torch.cuda.stream(cons):
        for _ in range(3):  # warm-up (allocator, autograd) before capture
            _step(bufs[0], ylong[0])
    torch.cuda.synchronize()
    for b in range(2):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cons):
            ylong[b].copy_(labs[b])
            _step(bufs[b], ylong[b])
        graphs[(bufs[b].data_ptr(), labs[b].data_ptr())] = g
    torch.cuda.synchronize()


def step_b(b, rows):
    if GRAPH and rows == B:
        graphs[(bufs[b].data_ptr(), labs[b].data_ptr())].replay()
    else:
        _step(bufs[b][:rows], labs[b][:rows].long())


def epoch_serial(e):
    L.set_stream(cons)  # the loader enqueues on the consumer's stream: no overlap
    L.epoch_permute(e, CHUNK, cons)
    with torch.cuda.stream(cons):
        for t in range(steps):
            rows = L.next_batch(bufs[0], labs[0], None, cons)
            step_b(0, rows)


ready = [torch.cuda.Event() for _ in range(2)]
free = [torch.cuda.Event() for _ in range(2)]
for ev in ready + free:  # materialise the events (torch creates them lazily at the first record)
    ev.record(cons)


def epoch_double(e, ctas=0):
    # the paper's double buffer: batch t+1 is assembled on the loader stream while step t runs on
    # the consumer stream; per-buffer events order the two (pp_next_batches_ev).  ctas > 0 caps
    # the gather grid so the consumer's kernels keep SMs while a batch is assembled.
    L.set_grid_limit(ctas)
    L.set_stream(loader_stream)
    L.epoch_permute(e, CHUNK, cons)
    rows = [0, 0]
    with torch.cuda.stream(cons):
        rows[0] = L.next_batches_ev(1, bufs[0], 0, labs[0], None, free[0], ready[0])[0]
        for t in range(steps):
            b, nb = t % 2, (t + 1) % 2
            if t + 1 < steps:
                rows[nb] = L.next_batches_ev(1, bufs[nb], 0, labs[nb], None, free[nb], ready[nb])[0]
            cons.wait_event(ready[b])
            step_b(b, rows[b])
            free[b].record(cons)
    L.set_grid_limit(0)


CTAS = int(os.environ.get("DB_CTAS", "16"))


def epoch_loader(e, ctas=0):
    # the loader alone (no consumer step), for the loader's own epoch time at this grid size
    L.set_grid_limit(ctas)
    L.set_stream(loader_stream)
    L.epoch_permute(e, CHUNK, cons)
    with torch.cuda.stream(cons):
        for t in range(steps):
            L.next_batches_ev(1, bufs[t % 2], 0, labs[t % 2], None, None, ready[t % 2])
        cons.wait_event(ready[(steps - 1) % 2])
    L.set_grid_limit(0)


def epoch_compute(e):
    with torch.cuda.stream(cons):
        for t in range(steps):
            step_b(0, B)


def timeit(fn):
    fn(0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(cons)
    for e in range(EPOCHS):
        fn(1 + e)
    b.record(cons)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / EPOCHS


res = {}
for name, fn in (("loader", epoch_loader), (f"loader_{CTAS}ctas", lambda e: epoch_loader(e, CTAS)),
                 ("compute", epoch_compute), ("serial", epoch_serial), ("double", epoch_double),
                 (f"double_{CTAS}ctas", lambda e: epoch_double(e, CTAS))):
    res[name] = timeit(fn)
    print(json.dumps({"placement": PLACEMENT, "chunk": CHUNK, "graph": GRAPH, "prio": os.environ.get("DB_LOADER_PRIO", "normal"),
                      "gather": os.environ.get("PPLOAD_GATHER", "auto"), "mode": name, "ms_per_epoch": res[name],
                      "nodes_per_s": N / res[name] * 1e3}), flush=True)
best = min(res["double"], res[f"double_{CTAS}ctas"])
print(json.dumps({"placement": PLACEMENT, "chunk": CHUNK, "graph": GRAPH, "double_buffer_speedup": res["serial"] / best,
                  "loader_hidden_fraction": (res["serial"] - best) / max(1e-9, res["serial"] - res["compute"]),
                  "paper": "1.33x GPU-resident (PAPER.md:441), 1.9x host-resident (PAPER.md:345), RTX A6000"}), flush=True)
L.close()
