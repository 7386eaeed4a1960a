#!/bin/bash
# CTA-pair (cta_group::2) fused linear: a first quick parity case, the kc suites, then an
# interleaved A/B of pairs vs single CTAs (debug bit 8192 flips the default)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 180 python -m pytest "tests/test_gpu_linear_kc.py::test_kc_cta_pair[3-256-0-512-300-tma-1]" -q -ra -x > gpurun_out/pytest_r2z.txt 2>&1
rc=$?
echo "first rc=$rc" >> gpurun_out/pytest_r2z.txt
if [ $rc -ne 0 ]; then exit 0; fi
timeout 900 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -ra -x >> gpurun_out/pytest_r2z.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2z.txt
LIN_AB=0,8192 timeout 900 python scripts/bench_linear_shapes.py > gpurun_out/lin_ab_pair.jsonl 2>> gpurun_out/lin_shapes.err
echo done
