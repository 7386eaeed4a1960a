"""One-off pin of the oracle casts over ALL 2^32 fp32 bit patterns (NaN excluded).

fp32->bf16 is compared with torch CPU ``.to(torch.bfloat16)``; fp32->fp16 with numpy
``astype(np.float16)``.  Calls only oracle/ and the two libraries.  Takes ~9 min on
8 cores; result recorded in DESIGN.md (run 2026-10-17: 0 mismatches).
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import oracle  # noqa: E402

t0 = time.time()
n = 1 << 26
bad_f16 = bad_bf16 = 0
for base in range(0, 1 << 32, n):
    b = np.arange(base, base + n, dtype=np.uint64).astype(np.uint32)
    f = b.view(np.float32)
    nan = np.isnan(f)
    with np.errstate(over="ignore"):
        ref16 = f.astype(np.float16).view(np.uint16)
    bad_f16 += int(((oracle.cast_f16(b) != ref16) & ~nan).sum())
    refbf = torch.from_numpy(f).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    bad_bf16 += int(((oracle.cast_bf16(b) != refbf) & ~nan).sum())
print(f"fp16 mismatches {bad_f16}, bf16 mismatches {bad_bf16}, {time.time() - t0:.0f}s")
sys.exit(1 if bad_f16 or bad_bf16 else 0)
