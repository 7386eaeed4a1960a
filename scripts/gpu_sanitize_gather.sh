#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $S --tool $tool --error-exitcode 9 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_gpu_edge_cases.py \
    -k "not products and not scale and not mag240m and not papers100m" > gpurun_out/sanitize_gather_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_gather_$tool.txt
done
