#!/bin/bash
# compute-sanitizer on the newest suites: compact store, DMA spill path, event double buffer, borrowed store,
# store propagation and the storage tier
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $S --tool $tool --error-exitcode 9 python -m pytest -q -x -m gpu tests/test_gpu_compact.py tests/test_gpu_dma_spill.py \
    tests/test_gpu_propagate_store.py tests/test_gpu_storage.py "tests/test_gpu_parity.py::test_event_double_buffer_matches_oracle" \
    "tests/test_gpu_parity.py::test_borrowed_device_store" -k "not ipc" > gpurun_out/sanitize_new_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_new_$tool.txt
done
echo done
