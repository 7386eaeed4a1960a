#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -ra -x > gpurun_out/pytest_r2n.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2n.txt
rm -f gpurun_out/lin_r2n.jsonl
for t in 0 1; do for pf in 0 1; do PPLOAD_LINEAR_TMA_A=$t PPLOAD_LINEAR_PREFETCH=$pf timeout 600 python scripts/bench_linear_shapes.py | sed "s/^{/{\"tma_a\": $t, \"pf\": $pf, /" >> gpurun_out/lin_r2n.jsonl 2>> gpurun_out/lin_shapes.err; done; done
echo done
