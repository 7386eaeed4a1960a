#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
rm -f gpurun_out/lin_dbg.jsonl
for d in 0 1 2 16 64 3 17 81 83; do PPLOAD_LINEAR_PREFETCH=0 PPLOAD_DEBUG_LINEAR=$d timeout 900 python scripts/bench_linear_shapes.py >> gpurun_out/lin_dbg.jsonl 2>> gpurun_out/lin_shapes.err; done
echo done
