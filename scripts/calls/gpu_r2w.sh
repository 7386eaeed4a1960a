#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -ra -x > gpurun_out/pytest_r2w.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2w.txt
PPLOAD_DEBUG_LINEAR=2048 timeout 600 python -m pytest tests/test_gpu_linear_kc.py -q -ra -x -k "mag or tma_gather4_sixteen" >> gpurun_out/pytest_r2w.txt 2>&1
echo "pytest2 rc=$?" >> gpurun_out/pytest_r2w.txt
LIN_AB=0,2048 LIN_SHAPES=mag240m timeout 900 python scripts/bench_linear_shapes.py > gpurun_out/lin_ab2.jsonl 2>> gpurun_out/lin_shapes.err
rm -f gpurun_out/lin_final.jsonl
for rep in 1 2; do timeout 900 python scripts/bench_linear_shapes.py >> gpurun_out/lin_final.jsonl 2>> gpurun_out/lin_shapes.err; done
echo done
