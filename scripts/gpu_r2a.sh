#!/bin/bash
# round-2 baseline: build, GPU tests, headline bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -ra -x > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 3 --skip-double-buffer --skip-next-rows > gpurun_out/bench.json 2> gpurun_out/bench.err
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1; nvidia-smi -q | head -80 > gpurun_out/smi.txt
echo done
