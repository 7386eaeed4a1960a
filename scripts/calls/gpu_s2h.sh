#!/bin/bash
# fused linear K-chunked at MAG240M rows: CTA pairs vs single CTAs -- interleaved A/B and source-level ncu captures
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s2h_build.txt 2>&1
LIN_AB=0,8192 LIN_SHAPES=mag240m,igb_large timeout 900 python scripts/bench_linear_shapes.py > $O/s2h_ab_pair.jsonl 2> $O/s2h.err
LIN_SHAPES=mag240m timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather_linear_kc -s 20 -c 1 -o $O/s2h_single python scripts/bench_linear_shapes.py > /dev/null 2>> $O/s2h.err
PPLOAD_LINEAR_PAIR=1 LIN_SHAPES=mag240m timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather_linear_kc -s 20 -c 1 -o $O/s2h_pair python scripts/bench_linear_shapes.py > /dev/null 2>> $O/s2h.err
echo done
