#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -ra -x > gpurun_out/pytest_r2p.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2p.txt
rm -f gpurun_out/lin_r2p.jsonl
for d in 0 64 16; do PPLOAD_DEBUG_LINEAR=$d timeout 600 python scripts/bench_linear_shapes.py >> gpurun_out/lin_r2p.jsonl 2>> gpurun_out/lin_shapes.err; done
echo done
