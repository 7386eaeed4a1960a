#!/bin/bash
# Fused-linear: per-tile timeline probe + one ncu --set full capture (source-level stalls).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 300 python scripts/ts_linear.py 0 2 > gpurun_out/ts_linear.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather_linear -s 5 -c 1 \
  -o gpurun_out/prof_linear python scripts/bench_linear.py > /dev/null 2> gpurun_out/ncu.err
echo "ncu rc=$?"
