"""§8(f)-1 consumer: fused batch assembly + per-hop linear on the tensor cores
(pp_next_batches_linear, tcgen05) against the oracle batch (O10) times W in float64.

Tolerance (derived, not fitted): bf16 x bf16 products are exact in fp32, so the only
fp32 error is in the K-1 additions of each dot product, |err| <= (K-1) * 2^-24 * sum|x w|
for any summation order; we allow 2 K 2^-24 sum|x w| (K = 128 padded, margin 2 for the
tensor core's internal adder tree).  A bf16 Z adds one RNE rounding, <= 2^-9 |Z|; we allow
2^-8 |Z| + the fp32 term."""
import numpy as np
import pytest

import oracle
from inputs import hop_tensor, node_set as make_node_set

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(autouse=True, params=["res", "auto"])
def kernel(request, monkeypatch):
    # every case on the W-resident kernel (PPLOAD_LINEAR=res) and on the default K-chunked one
    monkeypatch.setenv("PPLOAD_LINEAR", request.param)
    return request.param


@pytest.fixture(scope="module")
def pp():
    import __graft_entry__ as ge

    ge.build()
    import paper_2504_13266_b200 as pp

    return pp


def weights(seed, H, F, D):
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal((H, F, D)) / np.sqrt(F)).astype(np.float32)
    return oracle.cast_bf16(w.view(np.uint32))  # bf16 bits [H, F, D]


def check(Zgpu, zdt, batch_bits, wbits):
    Zref, S = oracle.hop_linear(batch_bits, wbits)
    tol = 2 * 128 * 2.0 ** -24 * S
    if zdt == "bf16":
        got = oracle.bf16_bits_to_f64(Zgpu.view(torch.int16).cpu().numpy().view(np.uint16))
        tol = tol + 2.0 ** -8 * np.abs(Zref)
    else:
        got = Zgpu.cpu().numpy().astype(np.float64)
    err = np.abs(got - Zref)
    bad = err > tol
    assert not bad.any(), f"{bad.sum()} of {bad.size} outside tolerance; worst excess {(err - tol).max()}"


@pytest.mark.parametrize("F,D,zdt", [(100, 512, "bf16"), (100, 256, "f32"), (128, 512, "f32"), (64, 256, "bf16"),
                                     (4, 512, "f32")])
def test_fused_linear_matches_oracle(pp, F, D, zdt):
    H, N, B = 4, 3001, 512
    X, hs, rs = hop_tensor(60 + F, H, N, F)
    S = make_node_set(61, N, 2500)
    wb = weights(62, H, F, D)
    Wd = torch.from_numpy(wb.view(np.int16).copy()).cuda().view(torch.bfloat16)
    tdt = torch.bfloat16 if zdt == "bf16" else torch.float32
    esz = 2 if zdt == "bf16" else 4
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                   node_set=S, batch_size=B, out_dtype=pp.PP_BF16) as L:
        L.epoch_permute(7, 16)
        order = oracle.epoch_order(7, S.shape[0], 16, node_set=S)
        steps = oracle.num_steps(S.shape[0], B)
        Z = torch.full((3, B, H, D), float("nan"), dtype=tdt, device="cuda")
        t = 0
        while t < steps:
            Z.fill_(float("nan"))
            rows = L.next_batches_linear(3, Wd, D, Z, zdt, B * H * D * esz)
            torch.cuda.synchronize()
            for i, nr in enumerate(rows):
                want, _, _ = oracle.batch(X.view(np.uint32), oracle.F32, hs, rs, H, F, order, B, 1, t + i, 0,
                                          oracle.BF16)
                assert nr == want.shape[0]
                check(Z[i, :nr], zdt, want, wb)
                if nr < B:  # rows past the ragged end are not written
                    assert torch.isnan(Z[i, nr:].float()).all()
            t += len(rows)
        assert L.next_batches_linear(1, Wd, D, Z, zdt, 0) == []


def test_fused_linear_products_shape(pp):
    # configs[1] row shape (F = 100, K = 3, B = 8192) with SIGN's hidden 512
    H, N, F, B, D = 4, 40_000, 100, 8192, 512
    with pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16) as L:
        L.fill_synthetic(2504)
        wb = weights(63, H, F, D)
        Wd = torch.from_numpy(wb.view(np.int16).copy()).cuda().view(torch.bfloat16)
        Z = torch.empty((1, B, H, D), dtype=torch.bfloat16, device="cuda")
        L.epoch_permute(9, 1)
        order = oracle.epoch_order(9, N, 1)
        for t in range(3):
            assert L.next_batches_linear(1, Wd, D, Z, "bf16", 0) == [B]
            torch.cuda.synchronize()
            rows = order[t * B:(t + 1) * B]
            sample = np.arange(0, B, 97)  # rows checked one by one against the oracle generator
            src = oracle.gen_rows(2504, oracle.F32, H, F, rows[sample])
            check(Z[0, sample], "bf16", oracle.cast_bf16(src), wb)


def test_fused_linear_rejects_unsupported(pp):
    H, N, F = 2, 500, 6
    X, hs, rs = hop_tensor(64, H, N, F)
    W = torch.zeros((H, F, 256), dtype=torch.bfloat16, device="cuda")
    Z = torch.zeros((64, H, 256), dtype=torch.bfloat16, device="cuda")
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                   batch_size=64, out_dtype=pp.PP_BF16) as L:
        L.epoch_permute(1, 1)
        with pytest.raises(pp.PPError) as ei:
            L.next_batches_linear(1, W, 256, Z, "bf16", 0)  # F % 4 != 0
        assert ei.value.status == pp.PP_ERR_INVALID
    X, hs, rs = hop_tensor(65, H, N, 8)
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=8, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                   batch_size=64, out_dtype=pp.PP_F32) as L:
        L.epoch_permute(1, 1)
        with pytest.raises(pp.PPError) as ei:
            L.next_batches_linear(1, W, 256, Z, "bf16", 0)  # fp32 batches: no 16-bit A operand
        assert ei.value.status == pp.PP_ERR_INVALID
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=8, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                   batch_size=64, out_dtype=pp.PP_BF16) as L:
        L.epoch_permute(1, 1)
        with pytest.raises(pp.PPError) as ei:
            L.next_batches_linear(1, W, 384, Z, "bf16", 0)  # D not in {256, 512}
        assert ei.value.status == pp.PP_ERR_INVALID


def test_fused_linear_weight_updates_between_calls(pp):
    # training semantics: W changes after every batch (optimizer step); each call must use the W it is
    # given (the kernel loads W_k by TMA at every launch, nothing is cached across calls); H = 3 leaves
    # one SM idle (grid = 147)
    H, N, F, B, D = 3, 2000, 48, 256, 256
    X, hs, rs = hop_tensor(66, H, N, F)
    with pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                   batch_size=B, out_dtype=pp.PP_BF16) as L:
        L.epoch_permute(3, 1)
        order = oracle.epoch_order(3, N, 1)
        Wd = torch.empty((H, F, D), dtype=torch.bfloat16, device="cuda")
        Z = torch.empty((1, B, H, D), dtype=torch.float32, device="cuda")
        for t in range(oracle.num_steps(N, B)):
            wb = weights(100 + t, H, F, D)
            Wd.copy_(torch.from_numpy(wb.view(np.int16).copy()).view(torch.bfloat16))  # in place, same pointer
            rows = L.next_batches_linear(1, Wd, D, Z, "f32", 0)
            torch.cuda.synchronize()
            want, _, _ = oracle.batch(X.view(np.uint32), oracle.F32, hs, rs, H, F, order, B, 1, t, 0, oracle.BF16)
            assert rows == [want.shape[0]]
            check(Z[0, :rows[0]], "f32", want, wb)
