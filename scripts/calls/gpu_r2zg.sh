#!/bin/bash
# A/B: gather4 issue from 8 warps (16-bit) and the register producers (fp32) vs the defaults
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
LIN_SHAPES=mag240m LIN_AB="0,E:PPLOAD_LINEAR_TMA_A=2,E:PPLOAD_LINEAR_TMA_A=0" timeout 900 python scripts/bench_linear_shapes.py > gpurun_out/lin_ab_g.jsonl 2>> gpurun_out/lin_shapes.err
LIN_SHAPES=igb_large LIN_AB="0,E:PPLOAD_LINEAR_TMA_F32=0" timeout 900 python scripts/bench_linear_shapes.py >> gpurun_out/lin_ab_g.jsonl 2>> gpurun_out/lin_shapes.err
echo done
