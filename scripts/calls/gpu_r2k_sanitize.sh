#!/bin/bash
# compute-sanitizer over the round-2 suites (all-to-all, fused linear K-chunked, review fixes,
# sliced propagation, timed path at reduced sizes, cuRAND pins)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
S=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_gpu_a2a.py tests/test_gpu_linear_kc.py tests/test_gpu_advice_r1.py tests/test_gpu_propagate_sliced.py tests/test_gpu_timed_path.py tests/test_gpu_curand_pins.py"
K="not 2449029 and not 111059956 and not products_three and not above_l2 and not oversized"
timeout 2400 $S --tool memcheck --error-exitcode 9 python -m pytest -q -m gpu $T -k "$K" > gpurun_out/r2_sanitize_memcheck.txt 2>&1
echo "memcheck rc=$?" >> gpurun_out/r2_sanitize_memcheck.txt
timeout 1800 $S --tool racecheck --error-exitcode 9 python -m pytest -q -m gpu tests/test_gpu_linear_kc.py tests/test_gpu_a2a.py -k "not above_l2" > gpurun_out/r2_sanitize_racecheck.txt 2>&1
echo "racecheck rc=$?" >> gpurun_out/r2_sanitize_racecheck.txt
timeout 1800 $S --tool synccheck --error-exitcode 9 python -m pytest -q -m gpu tests/test_gpu_linear_kc.py tests/test_gpu_a2a.py > gpurun_out/r2_sanitize_synccheck.txt 2>&1
echo "synccheck rc=$?" >> gpurun_out/r2_sanitize_synccheck.txt
echo done
