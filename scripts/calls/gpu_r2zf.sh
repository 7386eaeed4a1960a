#!/bin/bash
# fp32 gather4 halves converted in place (two chunks of staging in flight): parity, products A/B
# (resident kernel vs K-chunked), row shapes, ncu captures of the K-chunked kernel at IGB rows and
# the products shape
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -ra -x > gpurun_out/pytest_r2zf.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2zf.txt
LIN_K=8 LIN_ROUNDS=2 timeout 900 python scripts/bench_linear.py > gpurun_out/lin_products_ab3.jsonl 2>> gpurun_out/lin_shapes.err
LIN_AB=0 timeout 1200 python scripts/bench_linear_shapes.py > gpurun_out/lin_shapes_inplace.jsonl 2>> gpurun_out/lin_shapes.err
LIN_SHAPES=igb_large LIN_ROWS=1000000 timeout 600 ncu --set full --import-source on \
  --clock-control none -k regex:k_gather_linear_kc -s 4 -c 1 -o gpurun_out/kc_igb_large_f \
  python scripts/bench_linear_shapes.py > gpurun_out/ncu_kc_f.log 2>&1
PPLOAD_LINEAR=kc LIN_K=8 LIN_ROUNDS=1 timeout 600 ncu --set full --import-source on --clock-control none \
  -k regex:k_gather_linear_kc -s 4 -c 1 -o gpurun_out/kc_products_f python scripts/bench_linear.py >> gpurun_out/ncu_kc_f.log 2>&1
echo done
