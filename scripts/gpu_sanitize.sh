#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on small configs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
S=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_gpu_parity.py::test_tiny_epoch_bit_exact tests/test_gpu_parity.py::test_gather_paths tests/test_gpu_parity.py::test_order_matches_oracle tests/test_gpu_parity.py::test_order_large_buckets tests/test_gpu_parity.py::test_spill_tier_equals_oracle tests/test_gpu_parity.py::test_loopback_sharded_equals_oracle tests/test_gpu_parity.py::test_epoch_prefetch"
for tool in memcheck racecheck synccheck; do
  timeout 1800 $S --tool $tool --error-exitcode 9 --target-processes all python -m pytest -q -x -m gpu $T \
    > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.txt
done
echo done
