"""Per-kernel SASS evidence (no GPU needed): which Blackwell instructions each hot kernel of
libppload.so actually contains -- 128/256-bit loads and stores, bulk copies (UBLKCP), TMA
(UTMALDG / UTMASTG / UBLKPF), tcgen05 (UTCHMMA, LDTM, UTCBAR), fp64 (DMUL / DADD) -- from
cuobjdump -sass.  Writes a markdown table to stdout."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2504_13266_b200", "libppload.so")
PATTERNS = {
    "LDG.128": r"\bLDG\.E[.\w]*\.128\b", "LDG.256": r"\bLDG\.E[.\w]*\.256\b", "STG.128": r"\bSTG\.E[.\w]*\.128\b",
    "UBLKCP": r"\bUBLKCP\b", "UBLKPF": r"\bUBLKPF\b", "UTMALDG": r"\bUTMALDG\b", "UTMASTG": r"\bUTMASTG\b",
    "UTCHMMA": r"\bUTC\w*MMA\b", "LDTM": r"\bLDTM\b", "UTCBAR": r"\bUTCBAR\b", "F2F.BF16": r"\bF2F\w*BF16",
    "F2FP": r"\bF2FP\b", "SHFL": r"\bSHFL\b", "MATCH": r"\bMATCH\b", "DMUL": r"\bDMUL\b", "DADD": r"\bDADD\b",
    "ATOMG/REDG": r"\b(ATOMG|REDG|RED)\b", "SYNCS": r"\bSYNCS\b",
}
KERNELS = ["k_gather_vec", "k_gather_tma", "k_gather_scalar", "k_gather_linear", "k_gather_linear_kc", "k_bucket_rank",
           "k_scatter", "k_hist", "k_cta_sort", "k_chunk_expand", "k_spmm_rows_v4", "k_spmm_store_v4", "k_spmm_sliced",
           "k_stage_cast", "k_cast_records", "k_a2a_index", "k_a2a_counts", "k_a2a_unpack", "k_assemble_staged"]

out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = collections.OrderedDict()
cur = None
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
    elif cur is not None:
        funcs[cur].append(line)
demangled = {}
if funcs:
    names = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True, text=True).stdout.splitlines()
    demangled = dict(zip(funcs, names))
print("| kernel (instantiations) | " + " | ".join(PATTERNS) + " |")
print("|---|" + "---|" * len(PATTERNS))
for k in KERNELS:
    agg = collections.Counter()
    n = 0
    for f, lines in funcs.items():
        d = demangled.get(f, f)
        if re.search(rf"\bppl::{k}\b[<(]", d) or re.search(rf"\b{k}\b", d.split("(")[0].split("<")[0]):
            if d.split("(")[0].split("<")[0].split("::")[-1] != k:
                continue
            n += 1
            text = "\n".join(lines)
            for name, pat in PATTERNS.items():
                agg[name] += len(re.findall(pat, text))
    if n:
        print(f"| {k} ({n}) | " + " | ".join(str(agg[p]) for p in PATTERNS) + " |")
sys.stdout.flush()
