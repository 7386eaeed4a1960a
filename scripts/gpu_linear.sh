#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 300 python scripts/ts_linear.py 0 3 > gpurun_out/ts_linear.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear.py -q -ra > gpurun_out/pytest_linear.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_linear.txt
timeout 600 python scripts/bench_linear.py > gpurun_out/bench_linear.jsonl 2> gpurun_out/bench_linear.err
echo done
