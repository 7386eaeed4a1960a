"""§8(f)-1 consumer at every BASELINE row shape: the K-chunked fused gather + per-hop linear
(k_gather_linear_kc) -- F walked in chunks of 64 with W_k streamed by TMA per chunk, so F = 768
(MAG240M, fp16 store) and F = 1024 (IGB-large) work, as do spilled, sharded and compact stores.
Z[j, k, :] = X_k[v_j, :] @ W_k with X in the batch dtype (the O10 batch: bf16 / f16 cast of fp32
records, or the 16-bit records themselves) and W in that dtype ("learns R+1 weight matrices for each
hop"; hidden 512).  Checked against oracle.hop_linear (float64) with
the tolerance of tests/test_gpu_linear.py at K = F rounded up to the chunk: 16-bit products are exact
in fp32, then K - 1 fp32 additions (2 K 2^-24 sum|x w| allowed) and, for bf16 Z, one RNE rounding."""
import numpy as np
import pytest

import oracle
from inputs import hop_tensor, node_set as make_node_set

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TDT = {oracle.BF16: torch.bfloat16, oracle.F16: torch.float16}


@pytest.fixture(scope="module")
def pp():
    import __graft_entry__ as ge

    ge.build()
    import paper_2504_13266_b200 as pp

    return pp


def weights(seed, H, F, D, dt):
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal((H, F, D)) / np.sqrt(F)).astype(np.float32).view(np.uint32)
    return oracle.cast_bf16(w) if dt == oracle.BF16 else oracle.cast_f16(w)


def check(Zgpu, zdt, batch_bits, wbits, dt, F):
    Zref, S = oracle.hop_linear(batch_bits, wbits, dt)
    K = -(-F // 64) * 64
    tol = 2 * K * 2.0 ** -24 * S
    if zdt == "bf16":
        got = oracle.bf16_bits_to_f64(Zgpu.view(torch.int16).cpu().numpy().view(np.uint16))
        tol = tol + 2.0 ** -8 * np.abs(Zref)
    else:
        got = Zgpu.cpu().numpy().astype(np.float64)
    fin = np.isfinite(Zref)
    err = np.abs(got - Zref)
    bad = fin & ~(err <= tol)  # a NaN where the reference is finite fails too
    assert not bad.any(), f"{bad.sum()} of {bad.size} outside tolerance; worst excess {np.nanmax(err[fin] - tol[fin])}"
    assert not np.isfinite(got[~fin]).any(), "finite output where the reference overflows or is NaN"


def run_and_check(pp, L, bits, in_dt, hs, rs, H, F, D, order, B, out_dt, zdt, W=1, r=0, k=2, seed=70):
    wb = weights(seed, H, F, D, out_dt)
    Wd = torch.from_numpy(wb.view(np.int16).copy()).cuda().view(TDT[out_dt])
    tdt = torch.bfloat16 if zdt == "bf16" else torch.float32
    esz = 2 if zdt == "bf16" else 4
    steps = oracle.num_steps(order.shape[0], B, W)
    Z = torch.empty((k, B, H, D), dtype=tdt, device="cuda")
    t = 0
    while t < steps:
        Z.fill_(float("nan"))
        rows = L.next_batches_linear(k, Wd, D, Z, zdt, B * H * D * esz)
        torch.cuda.synchronize()
        for i, nr in enumerate(rows):
            want, _, _ = oracle.batch(bits, in_dt, hs, rs, H, F, order, B, W, t + i, r, out_dt)
            assert nr == want.shape[0]
            if nr:
                check(Z[i, :nr], zdt, want, wb, out_dt, F)
            if nr < B:
                assert torch.isnan(Z[i, nr:].float()).all()
        t += len(rows)


@pytest.mark.parametrize("F,D,out_dt,zdt", [(1024, 512, oracle.BF16, "bf16"), (768, 256, oracle.F16, "f32"),
                                            (136, 512, oracle.BF16, "f32"), (8, 256, oracle.F16, "bf16"),
                                            (200, 512, oracle.F16, "bf16")])
def test_kc_fp32_store(pp, F, D, out_dt, zdt):
    H, N, B = 3, 1500, 256
    X, hs, rs = hop_tensor(71 + F, H, N, F)
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                   batch_size=B, out_dtype=out_dt) as L:
        L.epoch_permute(4, 1)
        run_and_check(pp, L, X.view(np.uint32), oracle.F32, hs, rs, H, F, D, oracle.epoch_order(4, N, 1), B, out_dt, zdt)


@pytest.mark.parametrize("dt", [oracle.F16, oracle.BF16])
def test_kc_sixteen_bit_store_mag240m_rows(pp, dt):
    # configs[4] row shape: fp16 records of 4 x 768 copied into the A operand as they are
    H, N, F, B, D = 4, 1200, 768, 512, 512
    X, hs, rs = hop_tensor(72, H, N, F, dtype=np.uint16)
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=dt,
                   batch_size=B, out_dtype=dt) as L:
        L.epoch_permute(5, 8)
        run_and_check(pp, L, X, dt, hs, rs, H, F, D, oracle.epoch_order(5, N, 8), B, dt, "f32")


def test_kc_spilled_compact_store(pp):
    H, N, F, B, D = 3, 3000, 96, 200, 256
    X, hs, rs = hop_tensor(73, H, N, F)
    S = make_node_set(74, N, 2100)
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                   node_set=S, store_set_only=True, batch_size=B, out_dtype=pp.PP_BF16,
                   hbm_budget_bytes=700 * H * F * 4) as L:
        assert L.query()["rows_spill"] > 0
        L.epoch_permute(6, 16)
        order = oracle.epoch_order(6, S.shape[0], 16, node_set=S)
        run_and_check(pp, L, X.view(np.uint32), oracle.F32, hs, rs, H, F, D, order, B, oracle.BF16, "bf16")


@pytest.mark.parametrize("W", [2, 3])
def test_kc_sharded_loopback(pp, W):
    # every rank's batches (global permutation, slice r of each step) with rows read from the owners
    H, N, F, B, D = 2, 2500, 128, 160, 512
    X, hs, rs = hop_tensor(75, H, N, F)
    Ls = [pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                    batch_size=B, out_dtype=pp.PP_BF16, world_size=W, rank=r, peers=pp.PP_PEERS_LOOPBACK)
          for r in range(W)]
    pp.pp_link_loopback([L.h for L in Ls])
    try:
        order = oracle.epoch_order(7, N, 4)
        for r, L in enumerate(Ls):
            L.epoch_permute(7, 4)
            run_and_check(pp, L, X.view(np.uint32), oracle.F32, hs, rs, H, F, D, order, B, oracle.BF16, "f32",
                          W=W, r=r)
    finally:
        for L in Ls:
            L.close()


def test_kc_equals_resident_kernel(pp, monkeypatch):
    # F = 128 runs on the resident-W kernel by default; PPLOAD_LINEAR=kc forces the K-chunked one.
    # Both accumulate the same exact products in fp32 (orders may differ): each within tolerance
    H, N, F, B, D = 4, 2000, 128, 512, 512
    X, hs, rs = hop_tensor(76, H, N, F)
    for mode in ("", "kc"):
        monkeypatch.setenv("PPLOAD_LINEAR", mode)
        with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                       batch_size=B, out_dtype=pp.PP_BF16) as L:
            L.epoch_permute(8, 1)
            run_and_check(pp, L, X.view(np.uint32), oracle.F32, hs, rs, H, F, D, oracle.epoch_order(8, N, 1), B,
                          oracle.BF16, "bf16", k=3)


def test_kc_local_epoch(pp):
    # a locality-aware epoch (pp_epoch_permute_local) on a sharded loader: this rank's rows only
    H, N, F, B, D = 2, 3001, 64, 128, 256
    X, hs, rs = hop_tensor(77, H, N, F)
    Ls = [pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                    batch_size=B, out_dtype=pp.PP_BF16, world_size=2, rank=r, peers=pp.PP_PEERS_LOOPBACK)
          for r in range(2)]
    pp.pp_link_loopback([L.h for L in Ls])
    try:
        L = Ls[1]
        L.epoch_permute_local(9, 1)
        local = L.query()["local_rows"]
        order = oracle.epoch_order(9, local, 1) * 2 + 1
        run_and_check(pp, L, X.view(np.uint32), oracle.F32, hs, rs, H, F, D, order, B, oracle.BF16, "f32")
    finally:
        for L_ in Ls:
            L_.close()


@pytest.mark.parametrize("tma_a", ["1", "0"])
@pytest.mark.parametrize("dt,F,chunk", [(oracle.F16, 768, 1), (oracle.BF16, 128, 7), (oracle.F16, 192, 64)])
def test_kc_tma_gather4_sixteen_bit(pp, monkeypatch, tma_a, dt, F, chunk):
    # 16-bit records with F % 64 == 0 in HBM: the A chunks come straight from the store by TMA
    # tile::gather4 (PPLOAD_LINEAR_TMA_A=1, opt-in) or through the register-staged producers (0, default);
    # node set + ragged last step included
    monkeypatch.setenv("PPLOAD_LINEAR_TMA_A", tma_a)
    H, N, B, D = 3, 2500, 384, 256
    X, hs, rs = hop_tensor(78 + F, H, N, F, dtype=np.uint16)
    S = make_node_set(79, N, 2101)
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=dt,
                   node_set=S, batch_size=B, out_dtype=dt) as L:
        L.epoch_permute(10, chunk)
        order = oracle.epoch_order(10, S.shape[0], chunk, node_set=S)
        run_and_check(pp, L, X, dt, hs, rs, H, F, D, order, B, dt, "f32", k=3)


@pytest.mark.parametrize("tma_f32", ["1", "0", "2"])
@pytest.mark.parametrize("F,out_dt,chunk", [(128, oracle.BF16, 1), (192, oracle.F16, 33), (1024, oracle.BF16, 256)])
def test_kc_tma_gather4_fp32_staging(pp, monkeypatch, tma_f32, F, out_dt, chunk):
    # fp32 records with F % 64 == 0 in HBM: 32-element halves by TMA gather4 into the staging ring,
    # cast by four converter warps (PPLOAD_LINEAR_TMA_F32=1, default), whole 64-element chunks by
    # unswizzled 256-byte gather4 boxes (2), or the register producers (0)
    monkeypatch.setenv("PPLOAD_LINEAR_TMA_F32", tma_f32)
    monkeypatch.setenv("PPLOAD_LINEAR", "kc")
    H, N, B, D = 2, 2300, 320, 512
    X, hs, rs = hop_tensor(80 + F, H, N, F)
    S = make_node_set(81, N, 1901)
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                   node_set=S, batch_size=B, out_dtype=out_dt) as L:
        L.epoch_permute(11, chunk)
        order = oracle.epoch_order(11, S.shape[0], chunk, node_set=S)
        run_and_check(pp, L, X.view(np.uint32), oracle.F32, hs, rs, H, F, D, order, B, out_dt, "f32", k=3)


@pytest.mark.parametrize("pair", ["1", "0"])
@pytest.mark.parametrize("H,F,dt,D,B,path", [
    (3, 256, oracle.F32, 512, 300, "tma"),      # fp32 gather4 + converters; tiles whose peer half is empty
    (2, 768, oracle.F16, 512, 1000, "tma"),     # 16-bit gather4 straight into A
    (4, 200, oracle.F32, 256, 640, "regs"),     # register producers (F % 64 != 0), one accumulator
    (1, 128, oracle.BF16, 512, 4096, "regs"),   # many tiles per pair: both barrier parities, deep W ring
    (80, 64, oracle.F16, 512, 256, "tma"),      # H > 148 / 2: single CTAs whatever the setting
])
def test_kc_cta_pair(pp, monkeypatch, pair, H, F, dt, D, B, path):
    # CTA pairs (PPLOAD_LINEAR_PAIR=1, default): clusters of two, the leader issuing M = 256
    # tcgen05.mma.cta_group::2 over both CTAs' A stages and W halves; each CTA drains its own rows
    monkeypatch.setenv("PPLOAD_LINEAR_PAIR", pair)
    monkeypatch.setenv("PPLOAD_LINEAR", "kc")
    if path == "regs":
        monkeypatch.setenv("PPLOAD_LINEAR_TMA_A", "0")
        monkeypatch.setenv("PPLOAD_LINEAR_TMA_F32", "0")
    N = 700 if H >= 80 else 5003
    X, hs, rs = hop_tensor(100 + H + F, H, N, F, dtype=np.float32 if dt == oracle.F32 else np.uint16)
    out_dt = oracle.BF16 if dt == oracle.F32 else dt
    pdt = {oracle.F32: pp.PP_F32, oracle.F16: pp.PP_F16, oracle.BF16: pp.PP_BF16}[dt]
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pdt,
                   batch_size=B, out_dtype=out_dt) as L:
        L.epoch_permute(13, 1)
        order = oracle.epoch_order(13, N, 1)
        bits = X.view(np.uint32) if dt == oracle.F32 else X
        zdt = "bf16" if D == 512 else "f32"
        run_and_check(pp, L, bits, dt, hs, rs, H, F, D, order, B, out_dt, zdt, k=3)


@pytest.mark.parametrize("layout", ["hop_rows", "records", "padded"])
@pytest.mark.parametrize("pair", ["1", "0"])
@pytest.mark.parametrize("tma_f32", ["1", "0", "2"])
@pytest.mark.parametrize("F", [100, 36, 196])
def test_kc_fp32_f_not_multiple_of_64(pp, monkeypatch, pair, tma_f32, F, layout):
    # fp32 records with F % 64 != 0 (products F = 100; F % 8 != 0 too): the last K chunk is padded
    # with zeros -- the fp32 gather4 reads 32-element halves that run into the next hop, which the
    # converters must zero (Inf planted at the start of hop 1 would otherwise poison hop 0's sums:
    # 0 * Inf = NaN); F <= 128 keeps W_k resident in the W stages (<= 256 for pairs).
    # layout: the TMA map of (node, hop) rows whose K padding is the out-of-bounds zero fill (default),
    # the map of whole records (experiment bit 524288), or records padded to 128 B (PPLOAD_REC_ALIGN)
    monkeypatch.setenv("PPLOAD_LINEAR", "kc")
    monkeypatch.setenv("PPLOAD_LINEAR_PAIR", pair)
    monkeypatch.setenv("PPLOAD_LINEAR_TMA_F32", tma_f32)
    if layout == "records":
        monkeypatch.setenv("PPLOAD_DEBUG_LINEAR", "524288")
    elif layout == "padded":
        monkeypatch.setenv("PPLOAD_REC_ALIGN", "128")
    H, N, B, D = 3, 3001, 640, 512
    X, hs, rs = hop_tensor(120 + F, H, N, F)
    trap = np.random.default_rng(121).choice(N, 64, replace=False)
    X[1, trap, :4] = np.inf
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                   batch_size=B, out_dtype=pp.PP_BF16) as L:
        L.epoch_permute(14, 1)
        order = oracle.epoch_order(14, N, 1)
        run_and_check(pp, L, X.view(np.uint32), oracle.F32, hs, rs, H, F, D, order, B, oracle.BF16, "bf16", k=3)


@pytest.mark.parametrize("dt,F", [(oracle.F32, 256), (oracle.F32, 100), (oracle.F16, 192)])
def test_kc_half_chunk_experiment_layout(pp, monkeypatch, dt, F):
    # experiment bit 2048 (three half-chunk W stages, six A slots: three in-place fp32 slot pairs)
    # must stay exact even though it is not the default
    monkeypatch.setenv("PPLOAD_LINEAR", "kc")
    monkeypatch.setenv("PPLOAD_DEBUG_LINEAR", "2048")
    H, N, B, D = 2, 2600, 512, 512
    X, hs, rs = hop_tensor(130 + F, H, N, F, dtype=np.float32 if dt == oracle.F32 else np.uint16)
    out_dt = oracle.BF16 if dt == oracle.F32 else dt
    pdt = pp.PP_F32 if dt == oracle.F32 else pp.PP_F16
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pdt,
                   batch_size=B, out_dtype=out_dt) as L:
        L.epoch_permute(15, 7)
        order = oracle.epoch_order(15, N, 7)
        bits = X.view(np.uint32) if dt == oracle.F32 else X
        run_and_check(pp, L, bits, dt, hs, rs, H, F, D, order, B, out_dt, "bf16", k=3)


@pytest.mark.parametrize("W", [2, 3])
def test_kc_cta_pair_sharded_loopback(pp, monkeypatch, W):
    # CTA pairs over a sharded store (register producers resolving owner / local row per row)
    monkeypatch.setenv("PPLOAD_LINEAR_PAIR", "1")
    H, N, F, B, D = 3, 4001, 128, 384, 512
    X, hs, rs = hop_tensor(140 + W, H, N, F)
    Ls = [pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                    batch_size=B, out_dtype=pp.PP_BF16, world_size=W, rank=r, peers=pp.PP_PEERS_LOOPBACK)
          for r in range(W)]
    pp.pp_link_loopback([L.h for L in Ls])
    try:
        order = oracle.epoch_order(16, N, 1)
        for L in Ls:
            L.epoch_permute(16, 1)
        for r, L in enumerate(Ls):
            run_and_check(pp, L, X.view(np.uint32), oracle.F32, hs, rs, H, F, D, order, B, oracle.BF16, "bf16",
                          W=W, r=r, k=2)
    finally:
        for L in Ls:
            L.close()


@pytest.mark.parametrize("F,chunk", [(100, 1), (68, 1), (128, 9), (124, 1), (1024, 1), (196, 5), (256, 1)])
@pytest.mark.parametrize("prefetch", ["0", "1"])
def test_kc_fp32_whole_tile_boxes_and_prefetch(pp, monkeypatch, F, chunk, prefetch):
    # experiment bit 4194304: fp32 records with an even number of 64-element chunks in pairs, one 512-byte
    # gather4 box per row stages chunks 2c, 2c + 1 of a tile, converted in place into slots 2p and 2p + 2
    # (F % 64 != 0: the (node, hop) row map, zero fill past F); PPLOAD_LINEAR_PREFETCH=1:
    # the TMA producers pull the next unit's rows into L2. Inf at the next hop's start must not leak.
    monkeypatch.setenv("PPLOAD_LINEAR", "kc")
    monkeypatch.setenv("PPLOAD_LINEAR_PAIR", "1")
    monkeypatch.setenv("PPLOAD_DEBUG_LINEAR", "4194304")
    monkeypatch.setenv("PPLOAD_LINEAR_PREFETCH", prefetch)
    H, N, B, D = 3, 4099, 896, 512
    X, hs, rs = hop_tensor(140 + F, H, N, F)
    trap = np.random.default_rng(141).choice(N, 64, replace=False)
    X[1, trap, :4] = np.inf
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                   batch_size=B, out_dtype=pp.PP_BF16) as L:
        L.epoch_permute(16, chunk)
        order = oracle.epoch_order(16, N, chunk)
        run_and_check(pp, L, X.view(np.uint32), oracle.F32, hs, rs, H, F, D, order, B, oracle.BF16, "bf16", k=3)
