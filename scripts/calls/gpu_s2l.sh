#!/bin/bash
# CTA pairs at IGB-large rows (fp32 records: gather4 halves + converters): source-level ncu, pair vs single
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s2l_build.txt 2>&1
LIN_SHAPES=igb_large timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather_linear_kc -s 20 -c 1 -o $O/s2l_single python scripts/bench_linear_shapes.py > /dev/null 2>> $O/s2l.err
PPLOAD_LINEAR_PAIR=1 LIN_SHAPES=igb_large timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather_linear_kc -s 20 -c 1 -o $O/s2l_pair python scripts/bench_linear_shapes.py > /dev/null 2>> $O/s2l.err
echo done
