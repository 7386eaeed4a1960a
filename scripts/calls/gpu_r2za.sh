#!/bin/bash
# ncu captures (full + source) of the K-chunked fused linear at MAG240M rows: single CTAs and CTA pairs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
for mode in 0 1; do
  PPLOAD_LINEAR_PAIR=$mode LIN_SHAPES=mag240m LIN_ROWS=1000000 timeout 600 ncu --set full --import-source on \
    --clock-control none -k regex:k_gather_linear_kc -s 4 -c 1 -o gpurun_out/kc_mag_pair$mode \
    python scripts/bench_linear_shapes.py > gpurun_out/ncu_kc_pair$mode.log 2>&1
  PPLOAD_LINEAR_PAIR=$mode LIN_SHAPES=igb_large LIN_ROWS=1000000 timeout 600 ncu --set full --import-source on \
    --clock-control none -k regex:k_gather_linear_kc -s 4 -c 1 -o gpurun_out/kc_igb_pair$mode \
    python scripts/bench_linear_shapes.py >> gpurun_out/ncu_kc_pair$mode.log 2>&1
done
echo done
