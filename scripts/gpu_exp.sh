#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 600 python scripts/exp_l2hint.py > gpurun_out/exp_l2hint.jsonl 2> gpurun_out/exp_l2hint.err
echo done
