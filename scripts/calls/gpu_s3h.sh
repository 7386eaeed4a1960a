#!/bin/bash
# products shape: register producers vs TMA gather4 staging for fp32 records, full and A-side only (bit 2097216)
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3h_build.txt 2>&1
LIN_AB="0,E:PPLOAD_LINEAR_TMA_F32=0,E:PPLOAD_LINEAR_TMA_F32=0+PPLOAD_LINEAR_PAIR=1,2097216,E:PPLOAD_LINEAR_TMA_F32=0+PPLOAD_DEBUG_LINEAR=2097216,E:PPLOAD_LINEAR_TMA_F32=0+PPLOAD_LINEAR_PAIR=1+PPLOAD_DEBUG_LINEAR=2097216,E:PPLOAD_LINEAR_TMA_F32=1+PPLOAD_DEBUG_LINEAR=2097216" LIN_SHAPES=products timeout 900 python scripts/bench_linear_shapes.py > $O/s3h_ab.jsonl 2> $O/s3h.err
echo done
