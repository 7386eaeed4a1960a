#!/bin/bash
# products-shape ablation: is the accumulator drain (epilogue) the A-side bound? (bit 2097152: no drain)
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3g_build.txt 2>&1
LIN_AB="0,66,2097152,2097216,2" LIN_SHAPES=products timeout 900 python scripts/bench_linear_shapes.py > $O/s3g_ab.jsonl 2> $O/s3g.err
LIN_AB="0,2097152,2" LIN_SHAPES=mag240m timeout 900 python scripts/bench_linear_shapes.py >> $O/s3g_ab.jsonl 2>> $O/s3g.err
echo done
