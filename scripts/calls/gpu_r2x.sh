#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
PPLOAD_DEBUG_LINEAR=4096 timeout 600 python -m pytest tests/test_gpu_linear_kc.py -q -ra -x -k "fp32" > gpurun_out/pytest_r2x.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2x.txt
LIN_AB=0,4096 LIN_SHAPES=igb_large timeout 900 python scripts/bench_linear_shapes.py > gpurun_out/lin_ab3.jsonl 2>> gpurun_out/lin_shapes.err
LIN_AB=0,2048 LIN_SHAPES=mag240m timeout 900 python scripts/bench_linear_shapes.py >> gpurun_out/lin_ab3.jsonl 2>> gpurun_out/lin_shapes.err
echo done
