#!/bin/bash
# ring counters (no 64-bit division on the issue paths) + whole-chunk W boxes: kc parity, A/B pairs vs
# single CTAs, ncu captures of both at MAG240M rows
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -ra -x > gpurun_out/pytest_r2zb.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2zb.txt
LIN_AB=0,8192 timeout 900 python scripts/bench_linear_shapes.py > gpurun_out/lin_ab_ring.jsonl 2>> gpurun_out/lin_shapes.err
for mode in 0 1; do
  PPLOAD_LINEAR_PAIR=$mode LIN_SHAPES=mag240m LIN_ROWS=1000000 timeout 600 ncu --set full --import-source on \
    --clock-control none -k regex:k_gather_linear_kc -s 4 -c 1 -o gpurun_out/kc_mag_ring_pair$mode \
    python scripts/bench_linear_shapes.py > gpurun_out/ncu_kc_ring$mode.log 2>&1
done
echo done
