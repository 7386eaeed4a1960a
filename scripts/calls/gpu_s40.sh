#!/bin/bash
# products-shape breakdown after the relay change (bits: 2 no Z stores, 64 no MMAs, 2097152 no drain)
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s40_build.txt 2>&1
LIN_AB="0,2,64,66,2097152,2097216" LIN_SHAPES=products,igb_large timeout 1200 python scripts/bench_linear_shapes.py > $O/s40_ab.jsonl 2> $O/s40.err
echo done
