#!/bin/bash
# Fused-linear parity + variants on the products shape.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear.py -q -x -ra > gpurun_out/pytest_linear.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_linear.txt
tail -3 gpurun_out/pytest_linear.txt
timeout 300 python scripts/ts_linear.py 0 > gpurun_out/ts_linear.txt 2>&1
timeout 600 python scripts/bench_linear.py --debug ${1:-0,2,3} > gpurun_out/linexp.jsonl 2> gpurun_out/linexp.err
PPLOAD_LINEAR_PREFETCH=0 timeout 600 python scripts/bench_linear.py > gpurun_out/linexp_nopf.jsonl 2>> gpurun_out/linexp.err
cat gpurun_out/linexp.jsonl; echo "-- no L2 prefetch:"; head -1 gpurun_out/linexp_nopf.jsonl
tail -5 gpurun_out/linexp.err
