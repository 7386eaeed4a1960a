#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
rm -f gpurun_out/lin_dbg2.jsonl
for t in 1 0; do for d in 0 16 64 2 80 18; do PPLOAD_LINEAR_TMA_A=$t PPLOAD_DEBUG_LINEAR=$d LIN_SHAPES=mag240m timeout 600 python scripts/bench_linear_shapes.py | sed "s/^{/{\"tma_a\": $t, /" >> gpurun_out/lin_dbg2.jsonl 2>> gpurun_out/lin_shapes.err; done; done
echo done
