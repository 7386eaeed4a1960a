#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/linexp.jsonl
for pf in 1 2 3; do
  PPLOAD_NVCC_EXTRA="-DPPL_LIN_PFDIST=$pf" python -c "import __graft_entry__ as g; g.build(force=True)" > gpurun_out/build.txt 2>&1
  timeout 600 python -m pytest tests/test_gpu_linear.py -m gpu -q -x > gpurun_out/pytest_linexp_pf$pf.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_linexp_pf$pf.txt
  for k in 8 299; do
    LIN_K=$k timeout 600 python scripts/bench_linear.py 2>> gpurun_out/linexp.err | head -1 | sed "s/^{/{\"pf\": $pf, /" >> gpurun_out/linexp.jsonl
  done
  PPLOAD_DEBUG_LINEAR=6 LIN_K=299 timeout 600 python scripts/bench_linear.py 2>> gpurun_out/linexp.err | head -1 | sed "s/^{/{\"pf\": $pf, \"debug\": 6, /" >> gpurun_out/linexp.jsonl
done
python -c "import __graft_entry__ as g; g.build(force=True)" > gpurun_out/build.txt 2>&1
