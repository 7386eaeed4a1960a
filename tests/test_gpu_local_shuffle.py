"""§8(f)-4 locality-aware local shuffle (pp_epoch_permute_local) against the oracle: rank r's
epoch = oracle epoch order over its local_rows positions, mapped to global ids lr*W + r, sliced
in batches of B; every row read from the rank's own store (loopback shards on one GPU)."""
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
    import paper_2504_13266_b200 as pp

    return pp


@pytest.mark.parametrize("W,chunk", [(1, 1), (2, 1), (3, 5), (4, 64)])
def test_local_shuffle_equals_oracle(pp, W, chunk):
    H, N, F, B = 3, 4001, 32, 128
    X, hs, rs = hop_tensor(80, H, N, F)
    bits = X.view(np.uint32)
    kw = dict(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
              batch_size=B, out_dtype=pp.PP_BF16)
    if W > 1:
        Ls = [pp.Loader(world_size=W, rank=r, peers=pp.PP_PEERS_LOOPBACK, **kw) for r in range(W)]
    else:
        Ls = [pp.Loader(**kw)]
    try:
        seen = np.zeros(N, dtype=np.int64)
        for r, L in enumerate(Ls):  # no pp_link_loopback: local epochs never touch peers
            n_loc = L.query()["local_rows"]
            L.epoch_permute_local(100 + r, chunk)
            q = L.query()
            assert q["local_epoch"] == 1 and q["steps_per_epoch"] == -(-n_loc // B)
            want_order = oracle.epoch_order(100 + r, n_loc, chunk) * W + r
            assert np.array_equal(L.get_order(), want_order)
            out = torch.empty((B, H, F), dtype=torch.bfloat16, device="cuda")
            nodes = torch.empty(B, dtype=torch.int64, device="cuda")
            t = 0
            while (rows := L.next_batch(out, None, nodes)) >= 0:
                torch.cuda.synchronize()
                v = want_order[t * B:t * B + rows]
                assert np.array_equal(nodes[:rows].cpu().numpy(), v)
                want = oracle.gather_cast(bits, oracle.F32, hs, rs, H, F, v, oracle.BF16)
                got = out[:rows].view(torch.int16).cpu().numpy().view(np.uint16)
                assert np.array_equal(got, want)
                np.add.at(seen, v, 1)
                t += 1
        assert (seen == 1).all()  # the W local epochs together still cover every node once
    finally:
        for L in Ls:
            L.close()


def test_local_then_global_epochs(pp):
    # switching back to a global epoch restores the global step count and order
    H, N, F, B = 2, 3000, 16, 100
    X, hs, rs = hop_tensor(81, H, N, F)
    Ls = [pp.Loader(data=X, num_nodes=N, num_hops=H, feat_dim=F, hop_stride=hs, row_stride=rs, dtype=pp.PP_F32,
                    batch_size=B, out_dtype=pp.PP_BF16, world_size=2, rank=r, peers=pp.PP_PEERS_LOOPBACK)
          for r in range(2)]
    try:
        pp.pp_link_loopback([L.h for L in Ls])
        for L in Ls:
            L.epoch_permute_local(5, 1)
            L.epoch_permute(6, 1)
            q = L.query()
            assert q["local_epoch"] == 0 and q["steps_per_epoch"] == oracle.num_steps(N, B, 2)
            assert np.array_equal(L.get_order(), oracle.epoch_order(6, N, 1))
    finally:
        for L in Ls:
            L.close()
