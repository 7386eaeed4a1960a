#!/bin/bash
# compute-sanitizer on the store-propagation and storage-tier parity tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
S=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_gpu_propagate_store.py -k not_ipc tests/test_gpu_storage.py"
for tool in memcheck racecheck synccheck; do
  timeout 1500 $S --tool $tool --error-exitcode 9 python -m pytest -q -x -m gpu tests/test_gpu_propagate_store.py tests/test_gpu_storage.py -k "not ipc" \
    > gpurun_out/sanitize_new_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_new_$tool.txt
done
echo done
