#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_linear_kc.py -q -ra -x > gpurun_out/pytest_r2s.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2s.txt
rm -f gpurun_out/lin_r2s.jsonl
for t in 1 0; do for d in 0 64; do PPLOAD_LINEAR_TMA_F32=$t PPLOAD_DEBUG_LINEAR=$d LIN_SHAPES=igb_large timeout 600 python scripts/bench_linear_shapes.py | sed "s/^{/{\"tma_f32\": $t, /" >> gpurun_out/lin_r2s.jsonl 2>> gpurun_out/lin_shapes.err; done; done
echo done
