"""Regression tests for the round-1 code-review findings:

* a loader created from a CUDA-tensor source with W > 1 builds its exchange copy only after the
  store upload has landed (the upload runs on the legacy stream, the cast on the loader stream);
* the scalar gather (an `out` that is not 16-byte aligned) reads peer rows from the owner's
  exchange copy, which holds 16-bit elements, instead of misreading them as fp32;
* the storage tier's vector assembly honours the alignment of `out`;
* PPGF container files are refused instead of being misread;
* records too large for the gather kernels' 2^40 reciprocal division fail at create.
Every batch is compared with the oracle bit for bit (O9/O10)."""
import numpy as np
import pytest

import oracle
from inputs import hop_tensor

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def pp():
    import __graft_entry__ as ge

    ge.build()
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2504_13266_b200 as pp

    return pp


def _bits16(t):
    return t.detach().cpu().view(torch.int16).numpy().view(np.uint16)


def _loopback(pp, W, **kw):
    Ls = [pp.Loader(world_size=W, rank=r, peers=pp.PP_PEERS_LOOPBACK, **kw) for r in range(W)]
    pp.pp_link_loopback([L.h for L in Ls])
    return Ls


def _check_ranks(Ls, bits, hs, rs, H, F, order, B, misalign_elems=0):
    W = len(Ls)
    n = order.shape[0]
    for r, L in enumerate(Ls):
        buf = torch.empty(B * H * F + 8, dtype=torch.bfloat16, device="cuda")
        out = buf[misalign_elems: misalign_elems + B * H * F].view(B, H, F)  # 2-byte aligned only if misaligned
        for t in range(oracle.num_steps(n, B, W)):
            rows = L.next_batch(out)
            torch.cuda.synchronize()
            want, _, _ = oracle.batch(bits, oracle.F32, hs, rs, H, F, order, B, W, t, r, oracle.BF16)
            assert rows == want.shape[0]
            assert np.array_equal(_bits16(out[:rows]), want), (r, t)


@pytest.mark.parametrize("W", [2, 3])
def test_exchange_copy_from_device_source(pp, W):
    H, N, F, B = 4, 40_009, 64, 1024
    X, hs, rs = hop_tensor(81, H, N, F)
    Xd = torch.from_numpy(X).cuda()
    Ls = _loopback(pp, W, data=Xd, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs,
                   dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16)
    try:
        assert all(L.query()["exchange_cast"] == 1 for L in Ls)
        order = oracle.epoch_order(3, N, 1)
        for L in Ls:
            L.epoch_permute(3, 1)
        _check_ranks(Ls, X.view(np.uint32), hs, rs, H, F, order, B)
    finally:
        for L in Ls:
            L.close()


def test_scalar_gather_reads_peer_exchange_copy(pp):
    # a 2-byte aligned `out` forces the scalar kernel; half of every batch comes from the peer's
    # 16-bit exchange copy
    W, H, N, F, B = 2, 4, 3001, 56, 160
    X, hs, rs = hop_tensor(82, H, N, F)
    Ls = _loopback(pp, W, data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs,
                   dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16)
    try:
        assert all(L.query()["exchange_cast"] == 1 for L in Ls)
        order = oracle.epoch_order(4, N, 8)
        for L in Ls:
            L.epoch_permute(4, 8)
        _check_ranks(Ls, X.view(np.uint32), hs, rs, H, F, order, B, misalign_elems=1)
    finally:
        for L in Ls:
            L.close()


def test_storage_tier_unaligned_out(pp, tmp_path):
    H, N, F, B = 3, 2000, 32, 128
    hops = np.random.default_rng(83).standard_normal((H, N, F)).astype(np.float32)
    paths = []
    for k in range(H):
        p = tmp_path / f"hop{k}.bin"
        hops[k].tofile(p)
        paths.append(str(p))
    with pp.Loader(files=paths, num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B,
                   out_dtype=pp.PP_BF16) as L:
        L.epoch_permute(5, 64)
        order = oracle.epoch_order(5, N, 64)
        buf = torch.empty(B * H * F + 8, dtype=torch.bfloat16, device="cuda")
        out = buf[1: 1 + B * H * F].view(B, H, F)
        for t in range(oracle.num_steps(N, B)):
            rows = L.next_batch(out)
            torch.cuda.synchronize()
            want, _, _ = oracle.batch(hops.view(np.uint32), oracle.F32, N * F, F, H, F, order, B, 1, t, 0, oracle.BF16)
            assert np.array_equal(_bits16(out[:rows]), want), t


def test_ppgf_container_refused(pp, tmp_path):
    H, N, F = 2, 100, 8
    paths = []
    for k in range(H):
        p = tmp_path / f"hop{k}.ppgf"
        body = np.zeros((N + 1024, F), np.float32)
        raw = bytearray(body.tobytes())
        raw[:4] = b"PPGF"
        p.write_bytes(bytes(raw))
        paths.append(str(p))
    with pytest.raises(pp.PPError) as ei:
        pp.Loader(files=paths, num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=8,
                  out_dtype=pp.PP_BF16)
    assert ei.value.status == pp.PP_ERR_INVALID
    assert "PPGF" in str(ei.value)


def test_oversized_record_fails_at_create(pp):
    # H*F = 2^23 fp32 -> bf16: 2^19 vector slots per row; 128 * (2^19)^2 >= 2^40
    with pytest.raises(pp.PPError) as ei:
        pp.Loader(num_nodes=2, num_hops=1, feat_dim=1 << 23, dtype=pp.PP_F32, batch_size=2, out_dtype=pp.PP_BF16)
    assert ei.value.status == pp.PP_ERR_INVALID
    # a record that fits the vector path but not the scalar one: an unaligned `out` is refused per call
    F = 1 << 17  # vpr = 2^14: 128 * 2^28 < 2^40; scalar: 128 * 2^34 >= 2^40
    with pp.Loader(num_nodes=4, num_hops=1, feat_dim=F, dtype=pp.PP_F32, batch_size=2, out_dtype=pp.PP_BF16) as L:
        L.fill_synthetic(1)
        L.epoch_permute(1, 1)
        buf = torch.empty(2 * F + 8, dtype=torch.bfloat16, device="cuda")
        with pytest.raises(pp.PPError) as ei:
            L.next_batch(buf[1: 1 + 2 * F].view(2, 1, F))
        assert ei.value.status == pp.PP_ERR_INVALID
        assert L.next_batch(buf[: 2 * F].view(2, 1, F)) == 2  # aligned: fine, and the handle is not poisoned
        torch.cuda.synchronize()
        want = oracle.cast_bf16(oracle.gen_rows(1, oracle.F32, 1, F, L.get_order()[:2]))
        assert np.array_equal(_bits16(buf[: 2 * F].view(2, 1, F)), want)


def test_pdl_chain_guard_on_reused_slots(pp):
    # consumer stream == loader stream: consecutive gathers are chained by programmatic dependent
    # launch, except a launch that rewrites a slot the chain still writes
    N, H, F, B = 50_000, 4, 32, 1024
    with pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16) as L:
        L.fill_synthetic(1)
        st = torch.cuda.Stream()
        L.set_stream(st)
        bufs = [torch.empty((B, H, F), dtype=torch.bfloat16, device="cuda") for _ in range(2)]
        ring = torch.empty((6, B, H, F), dtype=torch.bfloat16, device="cuda")
        order = oracle.epoch_order(3, N, 1)
        with torch.cuda.stream(st):
            L.epoch_permute(3, 1, st)
            q0 = L.query()["pdl_launches"]
            for t in range(6):  # two buffers alternated: calls 2 and 4 reuse buffer 0 -> serialised
                L.next_batch(bufs[t % 2], None, None, st)
            q1 = L.query()["pdl_launches"]
            L.epoch_permute(3, 1, st)  # the epoch again: its first gather is serialised
            for t in range(6):  # six distinct slots: every launch after the first is chained
                L.next_batch(ring[t], None, None, st)
            q2 = L.query()["pdl_launches"]
        st.synchronize()
        assert q1 - q0 == 3 and q2 - q1 == 5, (q1 - q0, q2 - q1)
        for t in range(6):  # ring slot t holds batch t
            want = oracle.cast_bf16(oracle.gen_rows(1, oracle.F32, H, F, order[t * B:(t + 1) * B]))
            assert np.array_equal(_bits16(ring[t]), want), t
        assert np.array_equal(_bits16(bufs[1]), oracle.cast_bf16(oracle.gen_rows(1, oracle.F32, H, F, order[5 * B:6 * B])))
