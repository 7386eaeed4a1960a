#!/bin/bash
# ncu source captures of both fused-linear kernels at the products shape
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
LIN_K=8 LIN_ROUNDS=1 timeout 600 ncu --set full --import-source on --clock-control none \
  -k regex:"^k_gather_linear$" -s 4 -c 1 -o gpurun_out/res_products python scripts/bench_linear.py > gpurun_out/ncu_res.log 2>&1
ncu -i gpurun_out/res_products.ncu-rep --page raw --csv > /dev/null 2>> gpurun_out/ncu_res.log || \
LIN_K=8 LIN_ROUNDS=1 timeout 600 ncu --set full --import-source on --clock-control none \
  -k regex:"k_gather_linear[^_]" -s 4 -c 1 -o gpurun_out/res_products python scripts/bench_linear.py >> gpurun_out/ncu_res.log 2>&1
echo done
