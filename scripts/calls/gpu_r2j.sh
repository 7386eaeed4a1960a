#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -ra --durations=25 > gpurun_out/pytest_gpu_full.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.txt
echo done
