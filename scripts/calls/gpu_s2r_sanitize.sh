#!/bin/bash
# compute-sanitizer over the K-chunked fused linear after the CTA-pair rework (relaxed expect_tx, per-warp and relay
# arrivals, 8 A slots, (tile, hop) units) and the resident-W kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
S=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_gpu_linear_kc.py tests/test_gpu_linear.py"
timeout 2400 $S --tool memcheck --error-exitcode 9 python -m pytest -q -m gpu $T > gpurun_out/r2s3_sanitize_kc_memcheck.txt 2>&1
echo "memcheck rc=$?" >> gpurun_out/r2s3_sanitize_kc_memcheck.txt
timeout 2400 $S --tool racecheck --error-exitcode 9 python -m pytest -q -m gpu $T -k "cta_pair or not_multiple or column or equals_resident or tma" > gpurun_out/r2s3_sanitize_kc_racecheck.txt 2>&1
echo "racecheck rc=$?" >> gpurun_out/r2s3_sanitize_kc_racecheck.txt
timeout 2400 $S --tool synccheck --num-cuda-barriers 65536 --error-exitcode 9 python -m pytest -q -m gpu $T -k "cta_pair or not_multiple or equals_resident or tma" > gpurun_out/r2s3_sanitize_kc_synccheck.txt 2>&1
echo "synccheck rc=$?" >> gpurun_out/r2s3_sanitize_kc_synccheck.txt
echo done
