#!/bin/bash
# one asm block per chunk and accumulator (4 MMAs) vs per-MMA issue: parity + interleaved A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -ra -x > gpurun_out/pytest_r2zi.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2zi.txt
LIN_AB=0,32768 timeout 1200 python scripts/bench_linear_shapes.py > gpurun_out/lin_ab_mma4.jsonl 2>> gpurun_out/lin_shapes.err
echo done
