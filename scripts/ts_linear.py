"""Print the per-tile timestamp probe of the fused linear kernel (CTA 0), steady state."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__ as ge  # noqa: E402

ge.build()
import paper_2504_13266_b200 as pp  # noqa: E402

N, H, F, B, D = 2_449_029, 4, 100, 8192, 512
L = pp.Loader(num_nodes=N, num_hops=H, feat_dim=F, dtype=pp.PP_F32, batch_size=B, out_dtype=pp.PP_BF16)
L.fill_synthetic(2504)
W = torch.from_numpy((np.random.default_rng(0).standard_normal((H, F, D)) / 10).astype(np.float32)).cuda().to(
    torch.bfloat16)
Z = torch.empty((8, B, H, D), dtype=torch.bfloat16, device="cuda")
L.epoch_permute(1, 1)
for dbg in sys.argv[1:] or ["0"]:
    os.environ["PPLOAD_DEBUG_LINEAR"] = dbg
    print("debug", dbg, flush=True)
    for rep in range(3):
        os.environ.pop("PPLOAD_DEBUG_TS", None)
        if rep == 2:
            os.environ["PPLOAD_DEBUG_TS"] = "1"
        L.next_batches_linear(8, W, D, Z, "bf16", B * H * D * 2)
        torch.cuda.synchronize()
        if L.query()["cursor"] >= L.query()["steps_per_epoch"] - 8:
            L.epoch_permute(2, 1)
