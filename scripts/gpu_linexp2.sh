#!/bin/bash
# fused-linear epilogue grouping experiments: A stages x staging buffers x slices per fence round
mkdir -p gpurun_out; rm -f gpurun_out/linexp.jsonl
for cfg in "2 2 1" "1 4 2" "1 4 4" "2 2 2"; do
  set -- $cfg
  PPLOAD_NVCC_EXTRA="-DPPL_LIN_STAGES=$1 -DPPL_LIN_EPIBUFS=$2 -DPPL_LIN_GROUP=$3" python -c "import __graft_entry__ as g; g.build(force=True)" > gpurun_out/build.txt 2>&1
  timeout 600 python -m pytest tests/test_gpu_linear.py -m gpu -q -x > gpurun_out/pytest_linexp_$1_$2_$3.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_linexp_$1_$2_$3.txt
  for k in 1 8 299; do
    LIN_K=$k timeout 600 python scripts/bench_linear.py 2>> gpurun_out/linexp.err | head -1 | sed "s/^{/{\"stages\": $1, \"epibufs\": $2, \"group\": $3, /" >> gpurun_out/linexp.jsonl
  done
done
python -c "import __graft_entry__ as g; g.build(force=True)" > gpurun_out/build.txt 2>&1
