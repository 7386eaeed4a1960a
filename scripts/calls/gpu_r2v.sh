#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
rm -f gpurun_out/lin_final.jsonl
for rep in 1 2; do timeout 900 python scripts/bench_linear_shapes.py >> gpurun_out/lin_final.jsonl 2>> gpurun_out/lin_shapes.err; done
echo done
