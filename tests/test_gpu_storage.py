"""§8(f)-3: the storage tier (PP_MEM_FILES).  One raw [N][F] file per hop;
each step's rows are read from the files (one read per run of consecutive node ids and hop),
DMA'd and cast on the GPU.  Batches, labels and node ids must equal the oracle's (O8-O10)
bit for bit for every chunk size, dtype pair, node set, W, I/O mode and access pattern."""
import numpy as np
import pytest

import oracle
from inputs import node_set as make_node_set

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TORCH_DT = {oracle.BF16: torch.bfloat16, oracle.F16: torch.float16, oracle.F32: torch.float32}


@pytest.fixture(scope="module")
def pp():
    import __graft_entry__ as ge

    ge.build()
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2504_13266_b200 as pp

    return pp


def write_hops(tmp_path, hops):
    """hops: [H, N, F] array -> H files of raw [N][F]."""
    paths = []
    for k in range(hops.shape[0]):
        p = tmp_path / f"hop{k}.bin"
        np.ascontiguousarray(hops[k]).tofile(p)
        paths.append(str(p))
    return paths


def bits_of(t, dt):
    x = t.detach().cpu()
    if dt == oracle.F32:
        return x.view(torch.int32).numpy().view(np.uint32)
    return x.view(torch.int16).numpy().view(np.uint16)


def run_epoch(pp, L, hops_bits, in_dt, H, N_total, F, order, B, W, r, out_dt, labels=None, k=1, check_nodes=True):
    steps = oracle.num_steps(order.shape[0], B, W)
    s_out = 4 if out_dt == oracle.F32 else 2
    ring = torch.empty((k, B, H, F), dtype=TORCH_DT[out_dt], device="cuda")
    nodes = torch.empty((k, B), dtype=torch.int64, device="cuda")
    labs = torch.empty((k, B), dtype=torch.int32, device="cuda") if labels is not None else None
    t = 0
    while t < steps:
        rows = L.next_batches(k, ring, B * H * F * s_out, labs, nodes)
        torch.cuda.synchronize()
        for i, nr in enumerate(rows):
            want, wl, wn = oracle.batch(hops_bits, in_dt, N_total * F, F, H, F, order, B, W, t + i, r, out_dt, labels)
            assert nr == want.shape[0], (t + i, nr)
            assert np.array_equal(bits_of(ring[i, :nr], out_dt), want), (r, t + i)
            if check_nodes:
                assert np.array_equal(nodes[i, :nr].cpu().numpy(), wn), (r, t + i)
            if labels is not None:
                assert np.array_equal(labs[i, :nr].cpu().numpy(), wl), (r, t + i)
        t += len(rows)
    assert L.next_batch(ring[0]) == -1  # epoch exhausted
    return steps


@pytest.mark.parametrize("chunk", [1, 7, 64, 256, 3001])
@pytest.mark.parametrize("direct", ["1", "0"])
def test_chunks_bit_exact(pp, tmp_path, monkeypatch, chunk, direct):
    monkeypatch.setenv("PPLOAD_IO_DIRECT", direct)
    H, N, F, B = 4, 3001, 100, 256
    hops = np.random.default_rng(chunk).standard_normal((H, N, F)).astype(np.float32)
    labels = (np.arange(N) * 7 % 47).astype(np.int32)
    L = pp.Loader(files=write_hops(tmp_path, hops), num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32,
                  labels=labels, batch_size=B, out_dtype=pp.PP_BF16)
    q = L.query()
    assert q["storage_mode"] in (1, 2) and (direct == "1" or q["storage_mode"] == 2)
    for seed in (11, 12):
        L.epoch_permute(seed, chunk)
        order = oracle.epoch_order(seed, N, chunk)
        run_epoch(pp, L, hops.view(np.uint32), oracle.F32, H, N, F, order, B, 1, 0, oracle.BF16, labels)
    assert L.query()["storage_bytes_read"] >= 2 * N * H * F * 4
    L.close()


@pytest.mark.parametrize("in_dt,out_dt,F", [(oracle.F32, oracle.F16, 64), (oracle.F16, oracle.F16, 128),
                                            (oracle.F32, oracle.F32, 12), (oracle.F32, oracle.BF16, 7),
                                            (oracle.F16, oracle.F16, 5)])
def test_dtypes_and_scalar_rows(pp, tmp_path, in_dt, out_dt, F):
    # F = 7 / 5: rows are not 16-byte multiples -> the per-element assembly path
    H, N, B, chunk = 3, 1500, 100, 32
    rng = np.random.default_rng(F)
    if in_dt == oracle.F32:
        hops = rng.standard_normal((H, N, F)).astype(np.float32)
        bits = hops.view(np.uint32)
    else:
        bits = rng.integers(0, 1 << 16, (H, N, F), dtype=np.uint16)
        bits &= 0xFBFF  # no Inf/NaN exponents
        hops = bits.view(np.float16)
    L = pp.Loader(files=write_hops(tmp_path, hops), num_nodes=N, num_hops=H, feat_dim=F, dtype=in_dt, batch_size=B,
                  out_dtype=out_dt)
    L.epoch_permute(5, chunk)
    run_epoch(pp, L, bits, in_dt, H, N, F, oracle.epoch_order(5, N, chunk), B, 1, 0, out_dt, k=3)
    L.close()


def test_node_set_and_ring(pp, tmp_path):
    H, N, F, B = 2, 5000, 32, 128
    hops = np.random.default_rng(4).standard_normal((H, N, F)).astype(np.float32)
    S = make_node_set(3, N, 1777)
    L = pp.Loader(files=write_hops(tmp_path, hops), num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32,
                  node_set=S, batch_size=B, out_dtype=pp.PP_BF16)
    for chunk in (1, 16):
        L.epoch_permute(8, chunk)
        order = oracle.epoch_order(8, S.shape[0], chunk, S)
        run_epoch(pp, L, hops.view(np.uint32), oracle.F32, H, N, F, order, B, 1, 0, oracle.BF16, k=4)
    L.close()


@pytest.mark.parametrize("W", [2, 3])
def test_ranks_read_their_slices(pp, tmp_path, W):
    # file loaders shard nothing: rank r reads slice r of every step of the global epoch
    H, N, F, B, chunk = 4, 4099, 48, 96, 24
    hops = np.random.default_rng(W).standard_normal((H, N, F)).astype(np.float32)
    paths = write_hops(tmp_path, hops)
    order = oracle.epoch_order(21, N, chunk)
    for r in range(W):
        L = pp.Loader(files=paths, num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B,
                      out_dtype=pp.PP_BF16, world_size=W, rank=r)
        L.epoch_permute(21, chunk)
        run_epoch(pp, L, hops.view(np.uint32), oracle.F32, H, N, F, order, B, W, r, oracle.BF16, k=2)
        L.close()


def test_seek_prefetch_and_consumer_stream(pp, tmp_path):
    # the staged next step must be dropped by a seek / a new epoch; a consumer stream gets events
    H, N, F, B, chunk = 3, 2000, 64, 128, 64
    hops = np.random.default_rng(9).standard_normal((H, N, F)).astype(np.float32)
    L = pp.Loader(files=write_hops(tmp_path, hops), num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32,
                  batch_size=B, out_dtype=pp.PP_BF16)
    cons = torch.cuda.Stream()
    bufs = [torch.empty((B, H, F), dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    order = oracle.epoch_order(1, N, chunk)
    L.epoch_permute(1, chunk)
    for t in (0, 1):
        assert L.next_batch(bufs[t % 2], consumer_stream=cons) > 0
    L.seek(7)  # step 2 was staged: must not be served as step 7
    for t in (7, 8, 3):
        if t == 3:
            L.seek(3)
        rows = L.next_batch(bufs[t % 2], consumer_stream=cons)
        cons.synchronize()
        want, _, _ = oracle.batch(hops.view(np.uint32), oracle.F32, N * F, F, H, F, order, B, 1, t, 0, oracle.BF16)
        assert rows == want.shape[0]
        assert np.array_equal(bits_of(bufs[t % 2][:rows], oracle.BF16), want), t
    # a new epoch mid-way: the staged step of the old epoch must not leak
    L.epoch_permute(2, chunk)
    order2 = oracle.epoch_order(2, N, chunk)
    rows = L.next_batch(bufs[0])
    torch.cuda.synchronize()
    want, _, _ = oracle.batch(hops.view(np.uint32), oracle.F32, N * F, F, H, F, order2, B, 1, 0, 0, oracle.BF16)
    assert np.array_equal(bits_of(bufs[0][:rows], oracle.BF16), want)
    L.close()


def test_invalid_file_loaders(pp, tmp_path):
    H, N, F = 2, 100, 8
    hops = np.zeros((H, N, F), np.float32)
    paths = write_hops(tmp_path, hops)
    short = tmp_path / "short.bin"
    np.zeros((N - 1, F), np.float32).tofile(short)
    with pytest.raises(pp.PPError) as ei:  # file shorter than N rows
        pp.Loader(files=[paths[0], str(short)], num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=8,
                  out_dtype=pp.PP_BF16)
    assert ei.value.status == pp.PP_ERR_INVALID
    with pytest.raises(pp.PPError) as ei:  # missing file
        pp.Loader(files=[paths[0], str(tmp_path / "nope.bin")], num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32,
                  batch_size=8, out_dtype=pp.PP_BF16)
    assert ei.value.status == pp.PP_ERR_INVALID
    with pytest.raises(pp.PPError) as ei:  # file loaders never link peers
        pp.Loader(files=paths, num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=8,
                  out_dtype=pp.PP_BF16, world_size=2, rank=0, peers=pp.PP_PEERS_LOOPBACK)
    assert ei.value.status == pp.PP_ERR_INVALID
    L = pp.Loader(files=paths, num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=8,
                  out_dtype=pp.PP_BF16)
    for call in (lambda: L.fill_synthetic(1), lambda: L.epoch_permute_local(1, 1), lambda: L.read_store(0, 1)):
        with pytest.raises(pp.PPError) as ei:
            call()
        assert ei.value.status == pp.PP_ERR_INVALID
    L.close()



def test_epoch_iterator_over_files(pp, tmp_path):
    # the double-buffered iterator (per-buffer events) on the storage tier
    H, N, F, B, chunk = 3, 2500, 32, 128, 64
    hops = np.random.default_rng(55).standard_normal((H, N, F)).astype(np.float32)
    L = pp.Loader(files=write_hops(tmp_path, hops), num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32,
                  batch_size=B, out_dtype=pp.PP_BF16)
    order = oracle.epoch_order(5, N, chunk)
    got = []
    for x, _, v in L.epoch(5, chunk, depth=3, nodes=True):
        torch.cuda._sleep(10000)
        got.append((x.clone(), v.clone()))
    torch.cuda.synchronize()
    assert len(got) == oracle.num_steps(N, B)
    for t, (x, v) in enumerate(got):
        want, _, wn = oracle.batch(hops.view(np.uint32), oracle.F32, N * F, F, H, F, order, B, 1, t, 0, oracle.BF16)
        assert np.array_equal(bits_of(x, oracle.BF16), want), t
        assert np.array_equal(v.cpu().numpy(), wn), t
    L.close()
