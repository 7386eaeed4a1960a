#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear.py -q -ra -x > gpurun_out/pytest_linear.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_linear.txt
echo done
