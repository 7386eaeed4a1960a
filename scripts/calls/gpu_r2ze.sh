#!/bin/bash
# descriptor increments in the MMA loop: parity, row shapes A/B (warp-wide vs lane-0 issue), ncu
# source captures at both row shapes and the products shape (K-chunked, forced)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -ra -x > gpurun_out/pytest_r2ze.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2ze.txt
LIN_AB=0,16384 timeout 1200 python scripts/bench_linear_shapes.py > gpurun_out/lin_ab_desc.jsonl 2>> gpurun_out/lin_shapes.err
for shp in mag240m igb_large; do
  LIN_SHAPES=$shp LIN_ROWS=1000000 timeout 600 ncu --set full --import-source on \
    --clock-control none -k regex:k_gather_linear_kc -s 4 -c 1 -o gpurun_out/kc_${shp}_e \
    python scripts/bench_linear_shapes.py > gpurun_out/ncu_kc_e.log 2>&1
done
PPLOAD_LINEAR=kc LIN_K=8 LIN_ROUNDS=1 timeout 600 ncu --set full --import-source on --clock-control none \
  -k regex:k_gather_linear_kc -s 4 -c 1 -o gpurun_out/kc_products_e python scripts/bench_linear.py >> gpurun_out/ncu_kc_e.log 2>&1
LIN_K=8 LIN_ROUNDS=1 timeout 600 ncu --set full --import-source on --clock-control none \
  -k regex:"k_gather_linear\(" -s 4 -c 1 -o gpurun_out/res_products_e python scripts/bench_linear.py >> gpurun_out/ncu_kc_e.log 2>&1
echo done
