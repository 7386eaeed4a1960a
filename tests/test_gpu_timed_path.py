"""GPU parity on the exact path bench.py times ("reshuffle ... at
the start of each epoch").

* The prefetched permutation (pp_epoch_prefetch on the side stream, the bucket sort with its grid
  capped at PPLOAD_PREFETCH_CTAS CTAs, so every k_bucket_rank warp walks many buckets through its
  software-pipelined loop) is compared with oracle.epoch_order over consecutive epochs, for unit
  counts that take the bucket path (U > 4096), with the default permutation path (no PPLOAD_PERMUTE).
* bench.py's own epoch loop (bench.epoch_loop: permute -> prefetch -> k = 8 steps per
  pp_next_batches launch into the 299-slot ring, programmatic dependent launch between launches)
  at the products size, three consecutive epochs: the whole node-id stream equals the oracle order
  and sampled batches equal the oracle's generator + cast, element by element.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SEED0 = 250413266


@pytest.fixture(scope="module")
def pp():
    import __graft_entry__ as ge

    ge.build()
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2504_13266_b200 as pp

    return pp


def _bits16(t):
    return t.detach().cpu().view(torch.int16).numpy().view(np.uint16)


@pytest.mark.parametrize("cap", [1, 148, 0])
@pytest.mark.parametrize("N,chunk", [(5_000, 1), (300_001, 1), (2_449_029, 1), (111_059_956, 8192)])
def test_prefetched_order_matches_oracle(pp, monkeypatch, cap, N, chunk):
    monkeypatch.delenv("PPLOAD_PERMUTE", raising=False)
    monkeypatch.setenv("PPLOAD_PREFETCH_CTAS", str(cap))  # read at pp_loader_create
    U = -(-N // chunk)
    assert U > 4096  # the bucket sort, not the one-CTA sort
    epochs = 4 if (cap == 148 or N < 1_000_000) else 2
    if N > 100_000_000 and cap != 148:
        epochs = 1
    B = 8192
    with pp.Loader(num_nodes=N, num_hops=1, feat_dim=4, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16) as L:
        out = torch.empty((B, 1, 4), dtype=torch.bfloat16, device="cuda")
        L.epoch_permute(SEED0, chunk)
        for e in range(epochs):
            L.epoch_prefetch(SEED0 + e + 1, chunk)
            for _ in range(3):  # a few batches of the current epoch overlap the prefetch
                L.next_batch(out)
            L.epoch_permute(SEED0 + e + 1, chunk)  # switches to the prefetched order
            got = L.get_order()
            want = oracle.epoch_order(SEED0 + e + 1, N, chunk)
            assert np.array_equal(got, want), f"epoch {e + 1}: prefetched order (cap {cap}) differs from the oracle"
            del got, want


def test_bench_loop_products_three_epochs(pp):
    """bench.py's timed loop verbatim, plus the node-id ring, at the products size (configs[1])."""
    import bench

    cfg = bench.CONFIGS["products"]
    N, H, F, B, chunk = cfg["N"], cfg["H"], cfg["F"], cfg["B"], cfg["chunk"]
    L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16)
    try:
        L.fill_synthetic(bench.DATA_SEED)
        stream = torch.cuda.Stream()
        L.set_stream(stream)
        steps = L.query()["steps_per_epoch"]
        assert steps == oracle.num_steps(N, B) == 299
        slot_bytes = B * H * F * 2
        nslots = bench.ring_slots(steps, 8, slot_bytes)
        assert nslots == steps  # the bench ring holds the whole epoch
        ring = torch.empty((nslots, B, H, F), dtype=torch.bfloat16, device="cuda")
        slots = list(ring.unbind(0))
        node_ring = torch.full((nslots, B), -1, dtype=torch.int64, device="cuda")
        node_slots = list(node_ring.unbind(0))
        rng = np.random.default_rng(7)
        with torch.cuda.stream(stream):
            for e in range(3):
                ring.view(torch.int16).fill_(-1)
                bench.epoch_loop(L, SEED0 + e, SEED0 + e + 1, chunk, steps, slots, slot_bytes, 8, stream,
                                 node_slots=node_slots)
                stream.synchronize()
                order = oracle.epoch_order(SEED0 + e, N, chunk)
                got_nodes = node_ring.cpu().numpy().reshape(-1)
                last = N - (steps - 1) * B
                assert np.array_equal(got_nodes[: (steps - 1) * B], order[: (steps - 1) * B]), f"epoch {e}: node ids"
                assert np.array_equal(got_nodes[(steps - 1) * B: (steps - 1) * B + last], order[(steps - 1) * B:])
                check = sorted({0, 7, 8, steps - 1, *rng.integers(1, steps - 1, 4).tolist()})
                for t in check:
                    s, e_ = oracle.batch_range(N, B, 1, t, 0)
                    src = oracle.gen_rows(bench.DATA_SEED, oracle.F32, H, F, order[s:e_])
                    assert np.array_equal(_bits16(ring[t, : e_ - s]), oracle.cast_bf16(src)), f"epoch {e} step {t}"
    finally:
        L.close()
