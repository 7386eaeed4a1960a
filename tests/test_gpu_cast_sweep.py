"""The device cast against the oracle over ALL 2^32 fp32 bit patterns (Cast row:
"Device cvt.rn.bf16/f16.f32 must match the oracle on the same sweep"; north star: bit-exact
"including the round-to-nearest-even cast").  The oracle casts were pinned over the same 2^32 sweep
against torch CPU / numpy (scripts/verify_cast_exhaustive.py).

Each chunk of 2^28 consecutive patterns is a borrowed device store [2^18][1][1024] fp32 read by the
product gather (identity order: chunk = N, so row i of the batch is record i), through the C ABI;
the oracle casts the same patterns on the host (one thread per chunk, in parallel)."""
import concurrent.futures as cf
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CHUNK_BITS = 28
F = 1024


@pytest.fixture(scope="module")
def pp():
    import __graft_entry__ as ge

    ge.build()
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2504_13266_b200 as pp

    return pp


def test_device_cast_all_2_32_patterns(pp):
    n_chunk = 1 << CHUNK_BITS
    rows = n_chunk // F
    mism = {oracle.BF16: 0, oracle.F16: 0}
    first_bad = {}
    pool = cf.ThreadPoolExecutor(max_workers=max(2, min(8, os.cpu_count() or 2)))
    outs = {dt: torch.empty((rows, 1, F), dtype=torch.bfloat16 if dt == oracle.BF16 else torch.float16,
                            device="cuda") for dt in mism}
    for c in range(1 << (32 - CHUNK_BITS)):
        base = c << CHUNK_BITS
        pat = np.arange(base, base + n_chunk, dtype=np.uint64).astype(np.uint32)
        futs = {dt: pool.submit(oracle.cast_bf16 if dt == oracle.BF16 else oracle.cast_f16, pat) for dt in mism}
        store = torch.from_numpy(pat.view(np.int32)).cuda().view(rows, 1, F)
        for dt, out in outs.items():
            with pp.Loader(data=store, num_nodes=rows, num_hops=1, feat_dim=F, hop_stride=F, row_stride=F,
                           dtype=pp.PP_F32, batch_size=rows, out_dtype=dt, borrow_device_data=True) as L:
                L.epoch_permute(1, rows)  # chunk = N: the identity order
                assert L.next_batch(out) == rows
                torch.cuda.synchronize()
            got = out.view(torch.int16).cpu().numpy().view(np.uint16).ravel()
            want = futs[dt].result()
            bad = np.nonzero(got != want)[0]
            mism[dt] += int(bad.size)
            if bad.size and dt not in first_bad:
                first_bad[dt] = (hex(int(pat[bad[0]])), hex(int(got[bad[0]])), hex(int(want[bad[0]])))
        del store
    pool.shutdown()
    assert mism == {oracle.BF16: 0, oracle.F16: 0}, f"mismatches {mism}, first (pattern, device, oracle): {first_bad}"
