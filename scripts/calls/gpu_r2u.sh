#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
LIN_AB=0,2048 timeout 900 python scripts/bench_linear_shapes.py > gpurun_out/lin_ab.jsonl 2>> gpurun_out/lin_shapes.err
echo done
