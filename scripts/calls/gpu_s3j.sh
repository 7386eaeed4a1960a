#!/bin/bash
# fp32 64 < F <= 128 in pairs: one 512-B gather4 box per (node, hop) row (tma_f32 = 3): parity, products A/B
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3j_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -x -ra > $O/s3j_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s3j_pytest.txt
if grep -q "pytest rc=0" $O/s3j_pytest.txt; then
LIN_AB="0,4194304,2097216,4196368" LIN_SHAPES=products timeout 900 python scripts/bench_linear_shapes.py > $O/s3j_ab.jsonl 2> $O/s3j.err
fi
echo done
