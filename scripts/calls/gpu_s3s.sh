#!/bin/bash
# the A side alone (no drain, no MMAs: bit 2097216) in pairs vs single CTAs, at the three shapes
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3s_build.txt 2>&1
LIN_AB="2097216,E:PPLOAD_LINEAR_PAIR=0+PPLOAD_DEBUG_LINEAR=2097216,2097152,E:PPLOAD_LINEAR_PAIR=0+PPLOAD_DEBUG_LINEAR=2097152" LIN_SHAPES=products,mag240m,igb_large timeout 1200 python scripts/bench_linear_shapes.py > $O/s3s_ab.jsonl 2> $O/s3s.err
echo done
