#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/lin_k.jsonl
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
for dbg in 7 15 6 14 79; do PPLOAD_DEBUG_LINEAR=$dbg LIN_K=299 timeout 600 python scripts/bench_linear.py 2>> gpurun_out/lin_k.err | head -1 | sed "s/^{/{\"debug\": $dbg, /" >> gpurun_out/lin_k.jsonl; done
