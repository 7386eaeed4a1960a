#!/bin/bash
# W-resident K-chunked kernel + fp32 gather4 for F % 64 != 0: parity, products-shape A/B (resident
# kernel vs K-chunked), row shapes A/B pairs vs single
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -ra -x > gpurun_out/pytest_r2zc.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2zc.txt
LIN_K=8 timeout 900 python scripts/bench_linear.py > gpurun_out/lin_products_ab.jsonl 2>> gpurun_out/lin_shapes.err
PPLOAD_LINEAR_PAIR=1 LIN_K=8 LIN_ROUNDS=2 timeout 900 python scripts/bench_linear.py > gpurun_out/lin_products_ab_pair.jsonl 2>> gpurun_out/lin_shapes.err
echo done
