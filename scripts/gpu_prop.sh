#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_propagate.py -q -ra > gpurun_out/pytest_prop.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_prop.txt
timeout 600 python scripts/bench_propagate.py > gpurun_out/bench_prop.jsonl 2> gpurun_out/bench_prop.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_rows -s 1 -c 1 \
  -o gpurun_out/prof_spmm python scripts/bench_propagate.py > /dev/null 2>> gpurun_out/ncu.err
echo done
