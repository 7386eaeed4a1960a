#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -ra -x > gpurun_out/pytest_r2h.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2h.txt
rm -f gpurun_out/lin_pf.jsonl
for pf in 0 2 4 8; do PPLOAD_LINEAR_PREFETCH=$pf timeout 900 python scripts/bench_linear_shapes.py | sed "s/^{/{\"pf\": $pf, /" >> gpurun_out/lin_pf.jsonl 2>> gpurun_out/lin_shapes.err; done
echo done
