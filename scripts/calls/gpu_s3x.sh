#!/bin/bash
# ncu --set full of the default K-chunked kernel at IGB-large rows (fp32 wide gather4, pairs) for profiles/
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3x_build.txt 2>&1
LIN_SHAPES=igb_large timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_linear_kc -s 20 -c 1 -o $O/s3x_prof_kc_igb python scripts/bench_linear_shapes.py > /dev/null 2> $O/s3x.err
echo done
