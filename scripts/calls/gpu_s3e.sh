#!/bin/bash
# products-shape ablation of the K-chunked fused linear (bits: 2 no Z stores, 64 no MMAs, 16 no W loads)
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3e_build.txt 2>&1
LIN_AB="0,2,64,66,16" LIN_SHAPES=products timeout 900 python scripts/bench_linear_shapes.py > $O/s3e_ablation_products.jsonl 2> $O/s3e.err
echo done
