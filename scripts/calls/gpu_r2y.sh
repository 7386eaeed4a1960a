#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -ra -x > gpurun_out/pytest_r2y.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2y.txt
PPLOAD_DEBUG_LINEAR=2048 timeout 600 python -m pytest tests/test_gpu_linear_kc.py -q -ra -x >> gpurun_out/pytest_r2y.txt 2>&1
echo "pytest2 rc=$?" >> gpurun_out/pytest_r2y.txt
LIN_AB=0,2048 timeout 900 python scripts/bench_linear_shapes.py > gpurun_out/lin_ab4.jsonl 2>> gpurun_out/lin_shapes.err
PPLOAD_LINEAR_TMA_A=0 PPLOAD_LINEAR_TMA_F32=0 LIN_AB=0 timeout 900 python scripts/bench_linear_shapes.py > gpurun_out/lin_ab4_regs.jsonl 2>> gpurun_out/lin_shapes.err
echo done
