#!/bin/bash
# ncu --set full of the final fused-linear kernel at the products shape and IGB-large rows
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s43_build.txt 2>&1
LIN_SHAPES=products timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_linear_kc -s 20 -c 1 -o $O/s43_prof_kc_products python scripts/bench_linear_shapes.py > /dev/null 2> $O/s43.err
LIN_SHAPES=igb_large timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_linear_kc -s 20 -c 1 -o $O/s43_prof_kc_igb python scripts/bench_linear_shapes.py > /dev/null 2>> $O/s43.err
echo done
