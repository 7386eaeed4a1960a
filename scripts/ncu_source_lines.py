"""Warp-stall samples of one kernel per (outermost) source line.

ncu's source page gives samples per SASS address; nvdisasm -gi gives each instruction's inlining
chain.  This joins the two so that a barrier wait inside an inlined helper is charged to the line
that called it (which role waited on which barrier).

  python scripts/ncu_source_lines.py REPORT.ncu-rep CUBIN FUNCTION_MANGLED [top] [kernel_first_line]
"""
import collections
import csv
import io
import re
import subprocess
import sys

SRC = "paper_2504_13266_b200/csrc/linear.cu"
SRC_NAME = "/" + SRC.rsplit("/", 1)[-1]


def sass_lines(cubin, fn, min_line=0):
    """offset -> (source line, instruction).  The line is the outermost frame of the inlining chain,
    or, with min_line, the innermost frame at or after min_line (the kernel's own body: a lambda
    inlined into it is then charged to its own lines, a helper above the kernel to its caller)."""
    out = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True, check=True).stdout
    cur, chain, res, fresh = None, [], {}, False
    for ln in out.splitlines():
        if ln.startswith(".text."):
            cur = ln[len(".text."):].rstrip(":")
            continue
        if cur != fn:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)(.*)', ln)
        if m:
            if fresh:
                chain, fresh = [], False
            # innermost first, outermost last; frames in other files (CUDA headers) are skipped
            if m.group(1).endswith(SRC_NAME):
                chain.append(int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
        if m:
            fresh = True
            line = chain[-1] if chain else -1
            if min_line:
                line = next((x for x in chain if x >= min_line), line)
            res[int(m.group(1), 16)] = (line, m.group(2).strip().rstrip(";"))
    return res


def main():
    rep, cubin, fn = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    min_line = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    ia, isamp = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
    reasons = [(i, n[len("stall_"):]) for i, n in enumerate(hdr) if n.startswith("stall_") and "Not Issued" not in n]
    body = [r for r in rows[2:] if len(r) == len(hdr)]
    base = int(body[0][ia], 16)
    lines = sass_lines(cubin, fn, min_line)
    per = collections.Counter()
    ins = collections.defaultdict(collections.Counter)
    why = collections.defaultdict(collections.Counter)
    for r in body:
        off = int(r[ia], 16) - base
        s = int(r[isamp] or 0)
        line, op = lines.get(off, (-1, "?"))
        per[line] += s
        ins[line][op.split()[0] if op else "?"] += s
        for i, n in reasons:
            why[line][n] += int(r[i] or 0)
    tot = sum(per.values())
    src = open(SRC).read().splitlines()
    print(f"# {rep}: {tot} samples")
    for line, s in per.most_common(top):
        text = src[line - 1].strip()[:90] if 0 < line <= len(src) else ""
        top_ops = ", ".join(f"{o}:{c}" for o, c in ins[line].most_common(2))
        top_ops += " | " + ", ".join(f"{o}:{c}" for o, c in why[line].most_common(2))
        print(f"{s:7d} {100 * s / tot:5.1f}%  L{line:<5} {text}   [{top_ops}]")


if __name__ == "__main__":
    main()
