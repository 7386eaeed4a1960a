#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
rm -f gpurun_out/lin_r2q.jsonl
for rep in 1 2; do for d in 0 512 1024 1536; do PPLOAD_DEBUG_LINEAR=$d LIN_SHAPES=mag240m timeout 600 python scripts/bench_linear_shapes.py >> gpurun_out/lin_r2q.jsonl 2>> gpurun_out/lin_shapes.err; done; done
echo done
