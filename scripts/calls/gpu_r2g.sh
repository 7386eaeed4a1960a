#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -ra -x > gpurun_out/pytest_r2g.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2g.txt
timeout 900 python scripts/bench_linear_shapes.py > gpurun_out/lin_shapes.jsonl 2> gpurun_out/lin_shapes.err
LIN_ROWS=600000 LIN_SHAPES=igb_large timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_linear_kc -s 3 -c 1 -o gpurun_out/prof_linear_kc python scripts/bench_linear_shapes.py > /dev/null 2>> gpurun_out/ncu.err
echo done
