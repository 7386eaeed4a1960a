#!/bin/bash
# compute-sanitizer memcheck over the whole GPU suite except the full-size (products / MAG240M-scale) cases
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
S=/usr/local/cuda/bin/compute-sanitizer
timeout 2400 $S --tool memcheck --error-exitcode 9 python -m pytest -q -m gpu tests \
  -k "not products and not scale and not mag240m and not papers100m and not ipc" > gpurun_out/sanitize_all_memcheck.txt 2>&1
echo "memcheck rc=$?" >> gpurun_out/sanitize_all_memcheck.txt
