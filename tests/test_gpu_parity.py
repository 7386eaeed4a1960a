"""GPU parity: libppload.so (sm_100a kernels, called through the C ABI) against the
CPU oracle, element by element, bit-exact (the loader's result is
unique once the Philox stream, the argsort tie-break and the RNE cast are fixed)."""
import numpy as np
import pytest

import oracle
from inputs import bit_sweep, hop_tensor, integer_hops, labels as make_labels, node_set as make_node_set

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pp():
    import __graft_entry__ as ge

    ge.build()
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2504_13266_b200 as pp

    return pp


TORCH_DT = {oracle.F32: torch.float32, oracle.BF16: torch.bfloat16, oracle.F16: torch.float16}
NP_BITS = {oracle.F32: np.uint32, oracle.BF16: np.uint16, oracle.F16: np.uint16}
ORACLE_OF = {0: oracle.F32, 1: oracle.BF16, 2: oracle.F16}  # pp_dtype -> oracle code (same numbering)


def bits_of(t, dt):
    x = t.detach().cpu()
    if dt == oracle.F32:
        return x.view(torch.int32).numpy().view(np.uint32)
    return x.view(torch.int16).numpy().view(np.uint16)


def run_epoch(L, B, H, F, out_dt, with_labels=False, consumer=None):
    """All batches of one epoch through pp_next_batch -> list of (feat bits, labels, nodes)."""
    out = torch.empty((B, H, F), dtype=TORCH_DT[out_dt], device="cuda")
    lab = torch.empty(B, dtype=torch.int32, device="cuda") if with_labels else None
    nodes = torch.empty(B, dtype=torch.int64, device="cuda")
    res = []
    while True:
        rows = L.next_batch(out, lab, nodes, consumer)
        if rows < 0:
            break
        torch.cuda.synchronize()
        res.append((bits_of(out[:rows], out_dt).copy(), None if lab is None else lab[:rows].cpu().numpy(),
                    nodes[:rows].cpu().numpy()))
    return res


def check_epoch(got, X, in_dt, hs, rs, H, F, order, B, out_dt, lab=None, W=1, r=0):
    steps = oracle.num_steps(order.shape[0], B, W)
    assert len(got) == steps
    for t, (feat, glab, gnodes) in enumerate(got):
        want, wlab, wnodes = oracle.batch(X, in_dt, hs, rs, H, F, order, B, W, t, r, out_dt, lab)
        assert np.array_equal(gnodes, wnodes), f"step {t}: node ids differ"
        assert np.array_equal(feat, want), f"step {t}: features differ"
        if lab is not None:
            assert np.array_equal(glab, wlab), f"step {t}: labels differ"


# --------------------------------------------------------------------------- config 1 (tiny)
@pytest.fixture(scope="module")
def tiny():
    hops = oracle.tiny_hops()  # [4, 2708, 128] fp32 by oracle SpMM (A0 precondition)
    return hops, hops.view(np.uint32)


@pytest.mark.parametrize("chunk", [1, 64, 256])
@pytest.mark.parametrize("out_dt", [oracle.BF16, oracle.F16])
def test_tiny_epoch_bit_exact(pp, tiny, chunk, out_dt):
    hops, bits = tiny
    H, N, F = hops.shape
    B = 256
    lab = make_labels(1, N)
    with pp.Loader(data=hops, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=N * F, row_stride=F,
                   dtype=pp.PP_F32, labels=lab, batch_size=B, out_dtype=out_dt) as L:
        for e in range(2):
            seed = 250413266 + e
            L.epoch_permute(seed, chunk)
            order = oracle.epoch_order(seed, N, chunk)
            assert np.array_equal(L.get_order(), order)
            got = run_epoch(L, B, H, F, out_dt, with_labels=True)
            check_epoch(got, bits, oracle.F32, N * F, F, H, F, order, B, out_dt, lab)


# --------------------------------------------------------------------------- permutation
@pytest.mark.parametrize("N,chunk", [(1, 1), (2, 1), (2, 2), (5, 2), (19, 1), (20, 1), (28, 1), (100, 7),
                                     (1000, 1), (4097, 256), (65536, 1), (100_003, 8192), (1 << 20, 1),
                                     (1_000_001, 3)])
def test_order_matches_oracle(pp, N, chunk):
    with pp.Loader(num_nodes=N, num_hops=1, feat_dim=8, batch_size=64, out_dtype=pp.PP_BF16) as L:
        for seed in (0, 250413266, 2**64 - 1):
            L.epoch_permute(seed, chunk)
            assert np.array_equal(L.get_order(), oracle.epoch_order(seed, N, chunk)), (N, chunk, seed)


@pytest.mark.parametrize("delta", [-3, -6, -30])
def test_order_large_buckets(pp, delta):
    # fewer, larger buckets exercise the multi-tile rank path (delta=-30: one bucket)
    N = 20_000 if delta != -30 else 3_000
    with pp.Loader(num_nodes=N, num_hops=1, feat_dim=8, batch_size=64, out_dtype=pp.PP_BF16) as L:
        pp.pp_debug_set_sort_bits_delta(L.h, delta)
        for chunk in (1, 3):
            L.epoch_permute(77, chunk)
            assert np.array_equal(L.get_order(), oracle.epoch_order(77, N, chunk))


def test_order_products_scale(pp):
    N = 2_449_029
    with pp.Loader(num_nodes=N, num_hops=1, feat_dim=8, batch_size=8192, out_dtype=pp.PP_BF16) as L:
        for chunk in (1, 8192):
            L.epoch_permute(250413266, chunk)
            assert np.array_equal(L.get_order(), oracle.epoch_order(250413266, N, chunk))


def test_order_papers100m_chunked(pp):
    # config 3 shape: N = 111,059,956 with chunk reshuffling c = 8192 (U = 13,558 chunks)
    N = 111_059_956
    with pp.Loader(num_nodes=N, num_hops=1, feat_dim=8, batch_size=8192, out_dtype=pp.PP_BF16,
                   hbm_budget_bytes=1 << 20) as L:
        L.epoch_permute(250413266, 8192)
        got = L.get_order()
    want = oracle.epoch_order(250413266, N, 8192)
    assert np.array_equal(got, want)


# --------------------------------------------------------------------------- layouts, dtypes, paths
@pytest.mark.parametrize("layout", ["hop_major", "node_major"])
@pytest.mark.parametrize("H,F,out_dt", [(4, 100, oracle.BF16), (3, 8, oracle.F16), (2, 3, oracle.BF16),
                                        (1, 5, oracle.F16), (4, 16, oracle.F32), (3, 7, oracle.F32)])
def test_layouts_and_paths(pp, layout, H, F, out_dt):
    N, B = 3001, 200
    X, hs, rs = hop_tensor(5, H, N, F, layout)
    bits = X.view(np.uint32)
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                   batch_size=B, out_dtype=out_dt) as L:
        info = L.query()
        assert info["gather_path"] == (0 if (H * F) % 8 == 0 or (out_dt == oracle.F32 and (H * F) % 4 == 0) else 1)
        L.epoch_permute(11, 1)
        got = run_epoch(L, B, H, F, out_dt)
        check_epoch(got, bits, oracle.F32, hs, rs, H, F, oracle.epoch_order(11, N, 1), B, out_dt)


@pytest.mark.parametrize("dt", [oracle.F16, oracle.BF16])
@pytest.mark.parametrize("F", [768, 12, 5])
def test_sixteen_bit_store_copy(pp, dt, F):
    # MAG240M shape class: fp16 store -> fp16 batches (bit copy)
    H, N, B = 4, 2000, 256
    X, hs, rs = hop_tensor(6, H, N, F, "hop_major", dtype=np.uint16)
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=dt,
                   batch_size=B, out_dtype=dt) as L:
        L.epoch_permute(3, 16)
        got = run_epoch(L, B, H, F, dt)
        check_epoch(got, X, dt, hs, rs, H, F, oracle.epoch_order(3, N, 16), B, dt)


@pytest.mark.parametrize("out_dt", [oracle.BF16, oracle.F16])
def test_device_cast_matches_oracle_bit_sweep(pp, out_dt):
    # identity order (chunk = N) makes batch j row i exactly pattern i: device cvt.rn vs oracle O10,
    # including subnormals, ties, overflow, -0 and NaN (-> 0x7FFF)
    b = bit_sweep(1 << 22)
    F = 1024
    n = (b.shape[0] + F - 1) // F
    pad = np.zeros(n * F, np.uint32)
    pad[: b.shape[0]] = b
    X = pad.reshape(n, F)
    with pp.Loader(data=X, num_nodes=n, num_hops=1, feat_dim=F, hop_stride=0, row_stride=F, dtype=pp.PP_F32,
                   batch_size=n, out_dtype=out_dt) as L:
        L.epoch_permute(1, n)
        out = torch.empty((n, 1, F), dtype=TORCH_DT[out_dt], device="cuda")
        assert L.next_batch(out) == n
        torch.cuda.synchronize()
        got = bits_of(out, out_dt).ravel()
    want = oracle.cast_bf16(pad) if out_dt == oracle.BF16 else oracle.cast_f16(pad)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first {hex(pad[bad[0]])}: got {hex(got[bad[0]])} want {hex(want[bad[0]])}"


def test_node_set_and_labels(pp):
    H, N_total, F, B = 3, 5000, 16, 128
    X, hs, rs = hop_tensor(7, H, N_total, F)
    S = make_node_set(8, N_total, 1234)
    lab = make_labels(9, N_total)
    with pp.Loader(data=X, num_nodes=N_total, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs,
                   dtype=pp.PP_F32, node_set=S, labels=lab, batch_size=B, out_dtype=pp.PP_BF16) as L:
        for chunk in (1, 100):
            L.epoch_permute(21, chunk)
            order = oracle.epoch_order(21, S.shape[0], chunk, node_set=S)
            assert np.array_equal(L.get_order(), order)
            got = run_epoch(L, B, H, F, oracle.BF16, with_labels=True)
            check_epoch(got, X.view(np.uint32), oracle.F32, hs, rs, H, F, order, B, oracle.BF16, lab)


def test_epoch_column_sums_integer_features(pp):
    # invariant pin at the GPU: sum of all batches == column sums of X_k (exact, integer features)
    H, N, F, B = 4, 2708, 128, 256
    Xi = integer_hops(10, H, N, F)
    with pp.Loader(data=Xi, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=N * F, row_stride=F,
                   dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16) as L:
        L.epoch_permute(5, 64)
        out = torch.empty((B, H, F), dtype=torch.bfloat16, device="cuda")
        total = torch.zeros((H, F), dtype=torch.float64, device="cuda")
        seen = torch.zeros(N, dtype=torch.int64, device="cuda")
        nodes = torch.empty(B, dtype=torch.int64, device="cuda")
        while (rows := L.next_batch(out, None, nodes)) >= 0:
            total += out[:rows].double().sum(0)
            seen.index_add_(0, nodes[:rows], torch.ones(rows, dtype=torch.int64, device="cuda"))
        torch.cuda.synchronize()
    assert torch.equal(seen.cpu(), torch.ones(N, dtype=torch.int64))
    assert np.array_equal(total.cpu().numpy().astype(np.int64), Xi.astype(np.int64).sum(axis=1))


# --------------------------------------------------------------------------- config 2 (products) at full size
@pytest.fixture(scope="module")
def products(pp):
    N, H, F, B = 2_449_029, 4, 100, 8192
    L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16)
    L.fill_synthetic(2504)
    yield L, N, H, F, B
    L.close()


def test_products_fill_matches_oracle_generator(pp, products):
    L, N, H, F, B = products
    rows = np.array([0, 1, 2, 1_000_003, N - 1])
    got = np.stack([L.read_store(int(r), 1)[0] for r in rows]).view(np.uint32).reshape(len(rows), H, F)
    assert np.array_equal(got, oracle.gen_rows(2504, oracle.F32, H, F, rows))


@pytest.mark.parametrize("chunk", [1, 8192])
def test_products_sampled_batches(pp, products, chunk):
    # the launch configuration bench.py times (products, B = 8192, bf16 out); batches sampled,
    # each checked row by row against the oracle's own generator + cast
    L, N, H, F, B = products
    seed = 250413266
    L.epoch_permute(seed, chunk)
    order = oracle.epoch_order(seed, N, chunk)
    assert np.array_equal(L.get_order(), order)
    steps = oracle.num_steps(N, B)
    out = torch.empty((B, H, F), dtype=torch.bfloat16, device="cuda")
    nodes = torch.empty(B, dtype=torch.int64, device="cuda")
    check = {0, 1, 137, steps - 1}
    for t in range(steps):
        rows = L.next_batch(out, None, nodes)
        if t in check:
            torch.cuda.synchronize()
            s, e = oracle.batch_range(N, B, 1, t, 0)
            assert rows == e - s
            src = oracle.gen_rows(2504, oracle.F32, H, F, order[s:e])
            assert np.array_equal(nodes[:rows].cpu().numpy(), order[s:e])
            assert np.array_equal(bits_of(out[:rows], oracle.BF16), oracle.cast_bf16(src))
    assert L.next_batch(out) == -1


def test_products_next_batches_equals_next_batch(pp, products):
    L, N, H, F, B = products
    L.epoch_permute(42, 1)
    k = 5
    ring = torch.empty((k, B, H, F), dtype=torch.bfloat16, device="cuda")
    rows = L.next_batches(k, ring, B * H * F * 2)
    assert rows == [B] * k
    L.seek(0)
    one = torch.empty((B, H, F), dtype=torch.bfloat16, device="cuda")
    for i in range(k):
        assert L.next_batch(one) == B
        torch.cuda.synchronize()
        assert torch.equal(one.view(torch.int16), ring[i].view(torch.int16))
    L.seek(297)
    tail = L.next_batches(k, ring, B * H * F * 2)
    assert tail == [B, N - 298 * B]


# --------------------------------------------------------------------------- UVA spill tier
@pytest.mark.parametrize("budget_rows", [0, 1000, 2999])
def test_spill_tier_equals_oracle(pp, budget_rows):
    # rows beyond the HBM budget are read zero-copy from pinned host memory; the batches must be
    # identical to the oracle (and hence to the all-HBM tier)
    H, N, F, B = 4, 3001, 100, 256
    X, hs, rs = hop_tensor(12, H, N, F)
    rec = H * F * 4
    budget = -1 if budget_rows == 0 else budget_rows * rec
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                   batch_size=B, out_dtype=pp.PP_BF16, hbm_budget_bytes=budget) as L:
        info = L.query()
        assert info["rows_hbm"] == budget_rows and info["rows_spill"] == N - budget_rows
        L.epoch_permute(8, 1)
        got = run_epoch(L, B, H, F, oracle.BF16)
        check_epoch(got, X.view(np.uint32), oracle.F32, hs, rs, H, F, oracle.epoch_order(8, N, 1), B, oracle.BF16)


def test_spill_fill_synthetic(pp):
    H, N, F = 3, 4000, 32
    with pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, batch_size=512, out_dtype=pp.PP_BF16,
                   hbm_budget_bytes=1500 * H * F * 4) as L:
        L.fill_synthetic(2504)
        rows = np.array([0, 1499, 1500, 3999])
        got = np.stack([L.read_store(int(r), 1)[0] for r in rows]).view(np.uint32).reshape(4, H, F)
        assert np.array_equal(got, oracle.gen_rows(2504, oracle.F32, H, F, rows))


# --------------------------------------------------------------------------- sharded (loopback on one GPU)
@pytest.mark.parametrize("W", [2, 4, 8])
@pytest.mark.parametrize("chunk", [1, 64])
def test_loopback_sharded_equals_oracle(pp, W, chunk):
    # nodes sharded round-robin (owner = v mod W); each rank's batch of step t is its slice of the
    # global permutation (O9), read from the owners' stores through peer pointers
    H, N, F, B = 4, 5003, 64, 128
    X, hs, rs = hop_tensor(13, H, N, F)
    lab = make_labels(14, N)
    Ls = [pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                    labels=lab, batch_size=B, out_dtype=pp.PP_BF16, world_size=W, rank=r,
                    peers=pp.PP_PEERS_LOOPBACK) for r in range(W)]
    try:
        assert sum(L.query()["local_rows"] for L in Ls) == N
        pp.pp_link_loopback([L.h for L in Ls])
        order = oracle.epoch_order(31, N, chunk)
        for L in Ls:
            L.epoch_permute(31, chunk)
        outs = [run_epoch(L, B, H, F, oracle.BF16, with_labels=True) for L in Ls]
        for r in range(W):
            check_epoch(outs[r], X.view(np.uint32), oracle.F32, hs, rs, H, F, order, B, oracle.BF16, lab, W=W, r=r)
        # W-independence: concatenating the ranks' batches of each step = the W = 1 stream
        flat = np.concatenate([np.concatenate([outs[r][t][2] for r in range(W)]) for t in range(len(outs[0]))])
        assert np.array_equal(flat, order)
    finally:
        for L in Ls:
            L.close()


def test_loopback_with_spill(pp):
    W, H, N, F, B = 2, 3, 2001, 32, 100
    X, hs, rs = hop_tensor(15, H, N, F)
    Ls = [pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                    batch_size=B, out_dtype=pp.PP_F16, world_size=W, rank=r, peers=pp.PP_PEERS_LOOPBACK,
                    hbm_budget_bytes=300 * H * F * 4) for r in range(W)]
    try:
        pp.pp_link_loopback([L.h for L in Ls])
        order = oracle.epoch_order(2, N, 1)
        for L in Ls:
            L.epoch_permute(2, 1)
        for r, L in enumerate(Ls):
            check_epoch(run_epoch(L, B, H, F, oracle.F16), X.view(np.uint32), oracle.F32, hs, rs, H, F, order, B,
                        oracle.F16, W=W, r=r)
    finally:
        for L in Ls:
            L.close()


# --------------------------------------------------------------------------- streams, state, errors
def test_double_buffer_consumer_stream(pp, tiny):
    # the paper's double buffer: alternate two outputs, consume on another stream
    hops, bits = tiny
    H, N, F = hops.shape
    B = 256
    with pp.Loader(data=hops, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=N * F, row_stride=F,
                   dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16) as L:
        L.epoch_permute(99, 1)
        order = oracle.epoch_order(99, N, 1)
        cons = torch.cuda.Stream()
        bufs = [torch.empty((B, H, F), dtype=torch.bfloat16, device="cuda") for _ in range(2)]
        sums = []
        t = 0
        with torch.cuda.stream(cons):
            while True:
                rows = L.next_batch(bufs[t % 2], consumer_stream=cons)
                if rows < 0:
                    break
                torch.cuda._sleep(20000)  # slow consumer: the next fill must not overwrite early
                sums.append(bufs[t % 2][:rows].float().sum())
                t += 1
        torch.cuda.synchronize()
        for t, s in enumerate(sums):
            feat, _, _ = oracle.batch(bits, oracle.F32, N * F, F, H, F, order, B, 1, t, 0, oracle.BF16)
            want = (feat.astype(np.uint32) << 16).view(np.float32).astype(np.float32)
            assert abs(float(s) - float(torch.from_numpy(want).float().sum())) <= 1e-3 * max(1.0, abs(float(s)))


def test_state_errors_and_resume(pp):
    N, B = 1000, 100
    X, hs, rs = hop_tensor(16, 2, N, 8)
    with pp.Loader(data=X, num_nodes=N, num_hops=2, feat_dim=8, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                   batch_size=B, out_dtype=pp.PP_BF16) as L:
        out = torch.empty((B, 2, 8), dtype=torch.bfloat16, device="cuda")
        with pytest.raises(pp.PPError) as ei:
            L.next_batch(out)
        assert ei.value.status == pp.PP_ERR_STATE
        for bad in (0, N + 1):
            with pytest.raises(pp.PPError) as ei:
                L.epoch_permute(1, bad)
            assert ei.value.status == pp.PP_ERR_INVALID
        lab = torch.empty(B, dtype=torch.int32, device="cuda")
        L.epoch_permute(1, 1)
        with pytest.raises(pp.PPError) as ei:
            L.next_batch(out, lab)  # no labels in this loader
        assert ei.value.status == pp.PP_ERR_INVALID
        first = run_epoch(L, B, 2, 8, oracle.BF16)
        assert L.next_batch(out) == -1  # PP_END_OF_EPOCH
        # resume: (seed, chunk, cursor) reproduces the stream
        L.epoch_permute(1, 1)
        L.seek(4)
        again = run_epoch(L, B, 2, 8, oracle.BF16)
        for a, b in zip(first[4:], again):
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[2], b[2])


def test_drop_last(pp):
    N, B = 1050, 100
    X, hs, rs = hop_tensor(17, 1, N, 8)
    with pp.Loader(data=X, num_nodes=N, num_hops=1, feat_dim=8, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                   batch_size=B, out_dtype=pp.PP_BF16, drop_last=True) as L:
        L.epoch_permute(1, 1)
        got = run_epoch(L, B, 1, 8, oracle.BF16)
        assert [g[0].shape[0] for g in got] == [B] * 10


def test_epoch_prefetch(pp, tiny):
    # the next epoch's order computed ahead on the side stream == computing it at permute time
    hops, bits = tiny
    H, N, F = hops.shape
    B = 256
    with pp.Loader(data=hops, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=N * F, row_stride=F,
                   dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16) as L:
        L.epoch_permute(1, 1)
        L.epoch_prefetch(2, 1)
        first = run_epoch(L, B, H, F, oracle.BF16)  # epoch 1 unaffected by the pending prefetch
        check_epoch(first, bits, oracle.F32, N * F, F, H, F, oracle.epoch_order(1, N, 1), B, oracle.BF16)
        L.epoch_permute(2, 1)  # matches: switch to the prefetched order
        assert np.array_equal(L.get_order(), oracle.epoch_order(2, N, 1))
        L.epoch_prefetch(3, 64)
        L.epoch_permute(4, 16)  # does not match: computed afresh
        assert np.array_equal(L.get_order(), oracle.epoch_order(4, N, 16))
        got = run_epoch(L, B, H, F, oracle.BF16)
        check_epoch(got, bits, oracle.F32, N * F, F, H, F, oracle.epoch_order(4, N, 16), B, oracle.BF16)
        for e in range(5, 9):  # steady-state pipelining across epochs
            L.epoch_prefetch(e, 7)
            run_epoch(L, B, H, F, oracle.BF16)
            L.epoch_permute(e, 7)
            assert np.array_equal(L.get_order(), oracle.epoch_order(e, N, 7))


@pytest.mark.parametrize("mode", ["ldg", "tma"])
@pytest.mark.parametrize("case", ["bf16", "f16", "copy16", "spill", "loopback", "nodeset"])
def test_gather_paths(pp, mode, case, monkeypatch):
    # both vector kernels (register-staged LDG and bulk-copy TMA) against the oracle
    monkeypatch.setenv("PPLOAD_GATHER", mode)
    H, N, F, B = 4, 4099, 100, 512
    out_dt = {"f16": oracle.F16, "copy16": oracle.F16}.get(case, oracle.BF16)
    dt16 = case == "copy16"
    X, hs, rs = hop_tensor(50, H, N, F, "hop_major", dtype=np.uint16 if dt16 else np.float32)
    in_dt = oracle.F16 if dt16 else oracle.F32
    bits = X if dt16 else X.view(np.uint32)
    lab = make_labels(51, N)
    kw = dict(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=in_dt,
              batch_size=B, out_dtype=out_dt, labels=lab)
    W = 2 if case == "loopback" else 1
    S = make_node_set(52, N, 3001) if case == "nodeset" else None
    if case == "spill":
        kw["hbm_budget_bytes"] = 1500 * H * F * 4
    if S is not None:
        kw["node_set"] = S
    if W > 1:
        Ls = [pp.Loader(world_size=W, rank=r, peers=pp.PP_PEERS_LOOPBACK, **kw) for r in range(W)]
        pp.pp_link_loopback([L.h for L in Ls])
    else:
        Ls = [pp.Loader(**kw)]
    try:
        n = S.shape[0] if S is not None else N
        order = oracle.epoch_order(9, n, 32, node_set=S)
        for r, L in enumerate(Ls):
            L.epoch_permute(9, 32)
            # three steps per launch into a ring, then single steps
            steps = oracle.num_steps(n, B, W)
            ring = torch.empty((3, B, H, F), dtype=TORCH_DT[out_dt], device="cuda")
            labs = torch.empty((3, B), dtype=torch.int32, device="cuda")
            nodes = torch.empty((3, B), dtype=torch.int64, device="cuda")
            t = 0
            while t < steps:
                rows = L.next_batches(3, ring, B * H * F * 2, labs, nodes)
                torch.cuda.synchronize()
                for i, nr in enumerate(rows):
                    want, wl, wn = oracle.batch(bits, in_dt, hs, rs, H, F, order, B, W, t + i, r, out_dt, lab)
                    assert nr == want.shape[0]
                    assert np.array_equal(bits_of(ring[i, :nr], out_dt), want), (case, mode, t + i)
                    assert np.array_equal(labs[i, :nr].cpu().numpy(), wl)
                    assert np.array_equal(nodes[i, :nr].cpu().numpy(), wn)
                t += len(rows)
    finally:
        for L in Ls:
            L.close()


@pytest.mark.parametrize("tie_bits", [2, 6])
def test_order_rank_tie_fallback(pp, monkeypatch, tie_bits):
    # narrow the fast-path sub-key so 32-bit ties are frequent: the full (key, id) fallback must
    # reproduce the oracle exactly
    monkeypatch.setenv("PPLOAD_DEBUG_TIE_BITS", str(tie_bits))
    N = 300_007
    with pp.Loader(num_nodes=N, num_hops=1, feat_dim=8, batch_size=64, out_dtype=pp.PP_BF16) as L:
        for chunk in (1, 7):
            L.epoch_permute(5, chunk)
            assert np.array_equal(L.get_order(), oracle.epoch_order(5, N, chunk))


def test_order_mag240m_scale_properties(pp):
    # configs[4] size (U = 244,160,499 units, bucket bits = 24): the oracle's qsort is too slow to
    # run here, so the unique argsort is pinned by its defining properties, all computed by the
    # oracle's own key function: bijection, keys non-decreasing along the order, ids ascending on
    # equal keys
    N = 244_160_499
    with pp.Loader(num_nodes=N, num_hops=1, feat_dim=8, batch_size=8192, out_dtype=pp.PP_BF16,
                   hbm_budget_bytes=1 << 20) as L:
        L.epoch_permute(250413266, 1)
        order = L.get_order()
    seen = np.zeros(N, dtype=np.uint8)
    seen[order] = 1
    assert seen.all()
    del seen
    keys = oracle.unit_keys(250413266, N)[order]
    assert (keys[1:] >= keys[:-1]).all()  # uint64 comparisons
    ties = np.nonzero(keys[1:] == keys[:-1])[0]
    assert (order[ties + 1] > order[ties]).all()


@pytest.mark.parametrize("layout", ["hop_major", "node_major"])
def test_device_resident_source(pp, layout):
    # hop matrices handed over as CUDA tensors (PP_MEM_DEVICE): copied device-to-device into the store
    H, N, F, B = 3, 2500, 40, 300
    X, hs, rs = hop_tensor(70, H, N, F, layout)
    Xd = torch.from_numpy(X).cuda()
    with pp.Loader(data=Xd, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                   batch_size=B, out_dtype=pp.PP_BF16) as L:
        L.epoch_permute(4, 3)
        got = run_epoch(L, B, H, F, oracle.BF16)
        check_epoch(got, X.view(np.uint32), oracle.F32, hs, rs, H, F, oracle.epoch_order(4, N, 3), B, oracle.BF16)


def test_event_double_buffer_matches_oracle(pp, tiny):
    # pp_next_batches_ev: two buffers, per-buffer free / ready events, a consumer stream that copies
    # each batch out after waiting on its ready event -- every batch equals the oracle's
    X, bits = tiny
    H, N, F = X.shape
    B = 256
    L = pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=N * F, row_stride=F, dtype=pp.PP_F32,
                  batch_size=B, out_dtype=pp.PP_BF16)
    cons = torch.cuda.Stream()
    bufs = [torch.empty((B, H, F), dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    for ev in ready + free:
        ev.record(cons)
    steps = oracle.num_steps(N, B)
    got = torch.empty((steps, B, H, F), dtype=torch.bfloat16, device="cuda")
    L.epoch_permute(77, 1, cons)
    rows = [0, 0]
    with torch.cuda.stream(cons):
        rows[0] = L.next_batches_ev(1, bufs[0], 0, None, None, free[0], ready[0])[0]
        for t in range(steps):
            b, nb = t % 2, (t + 1) % 2
            if t + 1 < steps:
                rows[nb] = L.next_batches_ev(1, bufs[nb], 0, None, None, free[nb], ready[nb])[0]
            cons.wait_event(ready[b])
            torch.cuda._sleep(20000)  # a slow consumer: the next batch must not overwrite this one early
            got[t, :rows[b]].copy_(bufs[b][:rows[b]])
            free[b].record(cons)
    torch.cuda.synchronize()
    order = oracle.epoch_order(77, N, 1)
    for t in range(steps):
        want, _, _ = oracle.batch(bits, oracle.F32, N * F, F, H, F, order, B, 1, t, 0, oracle.BF16)
        assert np.array_equal(got[t, :want.shape[0]].cpu().view(torch.int16).numpy().view(np.uint16), want), t
    assert L.next_batches_ev(1, bufs[0], 0) == []
    L.close()


def test_borrowed_device_store(pp, tiny):
    # borrow_device_data: the caller's node-major device tensor is used in place (no copy);
    # batches equal the oracle's, writes through the loader land in the caller's tensor
    hops, bits = tiny
    H, N, F = hops.shape
    B = 256
    nm = torch.from_numpy(np.ascontiguousarray(hops.transpose(1, 0, 2))).cuda()  # [N, H, F] fp32
    with pp.Loader(data=nm, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=F, row_stride=H * F, dtype=pp.PP_F32,
                   batch_size=B, out_dtype=pp.PP_BF16, borrow_device_data=True) as L:
        order = oracle.epoch_order(12, N, 1)
        L.epoch_permute(12, 1)
        out = torch.empty((B, H, F), dtype=torch.bfloat16, device="cuda")
        for t in range(oracle.num_steps(N, B)):
            rows = L.next_batch(out)
            torch.cuda.synchronize()
            want, _, _ = oracle.batch(bits, oracle.F32, N * F, F, H, F, order, B, 1, t, 0, oracle.BF16)
            assert np.array_equal(out[:rows].cpu().view(torch.int16).numpy().view(np.uint16), want), t
        # in place: the loader's store is the caller's tensor
        L.fill_synthetic(2504)
        torch.cuda.synchronize()
        want = oracle.gen_rows(2504, oracle.F32, H, F, np.arange(5)).reshape(5, H * F)
        assert np.array_equal(nm[:5].reshape(5, H * F).cpu().view(torch.int32).numpy().view(np.uint32), want)
    # layouts that cannot be borrowed are refused
    with pytest.raises(pp.PPError) as ei:
        pp.Loader(data=torch.from_numpy(hops).cuda(), num_nodes=N, num_hops=H, feat_dim=F, hop_stride=N * F,
                  row_stride=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16, borrow_device_data=True)
    assert ei.value.status == pp.PP_ERR_INVALID
    with pytest.raises(pp.PPError) as ei:  # host data
        pp.Loader(data=hops, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=N * F, row_stride=F, dtype=pp.PP_F32,
                  batch_size=B, out_dtype=pp.PP_BF16, borrow_device_data=True)
    assert ei.value.status == pp.PP_ERR_INVALID


@pytest.mark.parametrize("depth,chunk", [(2, 1), (3, 64)])
def test_epoch_iterator_double_buffer(pp, tiny, depth, chunk):
    # Loader.epoch: the double-buffered iterator over pp_next_batches_ev; a slow consumer on the
    # current stream copies each yielded batch out; everything equals the oracle
    hops, bits = tiny
    H, N, F = hops.shape
    B = 256
    lab = make_labels(3, N)
    with pp.Loader(data=hops, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=N * F, row_stride=F, dtype=pp.PP_F32,
                   labels=lab, batch_size=B, out_dtype=pp.PP_BF16) as L:
        steps = oracle.num_steps(N, B)
        got = torch.empty((steps, B, H, F), dtype=torch.bfloat16, device="cuda")
        gl = torch.empty((steps, B), dtype=torch.int32, device="cuda")
        gv = torch.empty((steps, B), dtype=torch.int64, device="cuda")
        n = []
        for t, (x, y, v) in enumerate(L.epoch(21, chunk, depth=depth, labels=True, nodes=True)):
            torch.cuda._sleep(20000)
            got[t, :x.shape[0]].copy_(x)
            gl[t, :x.shape[0]].copy_(y)
            gv[t, :x.shape[0]].copy_(v)
            n.append(x.shape[0])
        torch.cuda.synchronize()
        assert len(n) == steps
        order = oracle.epoch_order(21, N, chunk)
        for t in range(steps):
            want, wl, wn = oracle.batch(bits, oracle.F32, N * F, F, H, F, order, B, 1, t, 0, oracle.BF16, lab)
            assert n[t] == want.shape[0]
            assert np.array_equal(got[t, :n[t]].cpu().view(torch.int16).numpy().view(np.uint16), want), t
            assert np.array_equal(gl[t, :n[t]].cpu().numpy(), wl) and np.array_equal(gv[t, :n[t]].cpu().numpy(), wn)


@pytest.mark.parametrize("gather", ["ldg", "tma"])
@pytest.mark.parametrize("ctas", [1, 3])
def test_grid_limit_bit_exact(pp, tiny, monkeypatch, gather, ctas):
    # pp_set_grid_limit: a 1- or 3-CTA persistent grid walks every tile of every step in a launch
    monkeypatch.setenv("PPLOAD_GATHER", gather)
    hops, bits = tiny
    H, N, F = hops.shape
    B = 256
    with pp.Loader(data=hops, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=N * F, row_stride=F, dtype=pp.PP_F32,
                   batch_size=B, out_dtype=pp.PP_BF16) as L:
        L.set_grid_limit(ctas)
        L.epoch_permute(31, 4)
        order = oracle.epoch_order(31, N, 4)
        steps = oracle.num_steps(N, B)
        ring = torch.empty((steps, B, H, F), dtype=torch.bfloat16, device="cuda")
        rows = L.next_batches(steps, ring, B * H * F * 2)
        torch.cuda.synchronize()
        assert len(rows) == steps
        for t, nr in enumerate(rows):
            want, _, _ = oracle.batch(bits, oracle.F32, N * F, F, H, F, order, B, 1, t, 0, oracle.BF16)
            assert np.array_equal(ring[t, :nr].cpu().view(torch.int16).numpy().view(np.uint16), want), t
        with pytest.raises(pp.PPError):
            L.set_grid_limit(-1)
