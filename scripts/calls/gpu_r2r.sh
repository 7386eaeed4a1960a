#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
S=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $S --tool memcheck --error-exitcode 9 python -m pytest -q -m gpu tests/test_gpu_linear_kc.py > gpurun_out/r2_sanitize_kc_memcheck.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_sanitize_kc_memcheck.txt
timeout 1200 $S --tool racecheck --error-exitcode 9 python -m pytest -q -m gpu tests/test_gpu_linear_kc.py > gpurun_out/r2_sanitize_kc_racecheck.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_sanitize_kc_racecheck.txt
timeout 1200 $S --tool synccheck --error-exitcode 9 python -m pytest -q -m gpu tests/test_gpu_linear_kc.py > gpurun_out/r2_sanitize_kc_synccheck.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_sanitize_kc_synccheck.txt
timeout 900 python scripts/bench_loopback.py > gpurun_out/loopback_peer.jsonl 2>> gpurun_out/loopback.err
LOOPBACK_EXCHANGE=a2a timeout 900 python scripts/bench_loopback.py > gpurun_out/loopback_a2a.jsonl 2>> gpurun_out/loopback.err
echo done
