#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -ra -x > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python scripts/exp_gather.py > gpurun_out/exp_gather.jsonl 2> gpurun_out/exp_gather.err
echo done
