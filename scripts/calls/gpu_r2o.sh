#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -ra -x > gpurun_out/pytest_r2o.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2o.txt
PPLOAD_LINEAR_TMA_A=2 timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -ra -x -k "tma or mag" >> gpurun_out/pytest_r2o.txt 2>&1
echo "pytest2 rc=$?" >> gpurun_out/pytest_r2o.txt
rm -f gpurun_out/lin_r2o.jsonl
for t in 1 2; do for d in 0 16 64 2; do PPLOAD_LINEAR_TMA_A=$t PPLOAD_DEBUG_LINEAR=$d LIN_SHAPES=mag240m timeout 600 python scripts/bench_linear_shapes.py | sed "s/^{/{\"tma_a\": $t, /" >> gpurun_out/lin_r2o.jsonl 2>> gpurun_out/lin_shapes.err; done; done
echo done
