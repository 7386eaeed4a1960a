#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -ra -x > gpurun_out/pytest_r2l.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2l.txt
rm -f gpurun_out/lin_tma.jsonl
for t in 1 0; do PPLOAD_LINEAR_TMA_A=$t LIN_SHAPES=mag240m timeout 900 python scripts/bench_linear_shapes.py | sed "s/^{/{\"tma_a\": $t, /" >> gpurun_out/lin_tma.jsonl 2>> gpurun_out/lin_shapes.err; done
LIN_SHAPES=mag240m timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_linear_kc -s 20 -c 1 -o gpurun_out/prof_linear_kc_tma python scripts/bench_linear_shapes.py > /dev/null 2>> gpurun_out/ncu.err
echo done
