#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 600 python scripts/exp_prefetch.py > gpurun_out/exp_prefetch.jsonl 2> gpurun_out/exp_prefetch.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_permute_paths.py -q -x > gpurun_out/pytest_gpu.txt 2>&1
echo done
