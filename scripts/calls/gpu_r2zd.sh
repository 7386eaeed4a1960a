#!/bin/bash
# warp-wide MMA issue (elect.sync) vs one lane; pairs off by default: parity, products A/B, row shapes A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -ra -x > gpurun_out/pytest_r2zd.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2zd.txt
LIN_K=8 LIN_ROUNDS=2 timeout 900 python scripts/bench_linear.py > gpurun_out/lin_products_ab2.jsonl 2>> gpurun_out/lin_shapes.err
LIN_AB=0,16384,8192 timeout 1200 python scripts/bench_linear_shapes.py > gpurun_out/lin_ab_elect.jsonl 2>> gpurun_out/lin_shapes.err
echo done
