#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/lin_k.jsonl
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_linear.py -m gpu -q -x > gpurun_out/pytest_linear.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_linear.txt
for k in 1 8 299; do LIN_K=$k timeout 600 python scripts/bench_linear.py 2>> gpurun_out/lin_k.err | head -1 >> gpurun_out/lin_k.jsonl; done
for dbg in 2; do PPLOAD_DEBUG_LINEAR=$dbg LIN_K=299 timeout 600 python scripts/bench_linear.py 2>> gpurun_out/lin_k.err | head -1 | sed "s/^{/{\"debug\": $dbg, /" >> gpurun_out/lin_k.jsonl; done
