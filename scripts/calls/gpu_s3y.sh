#!/bin/bash
# relay lane: default-semantics remote arrival instead of release.cluster (bit 67108864): parity, A/B
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3y_build.txt 2>&1
PPLOAD_DEBUG_LINEAR=67108864 timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -x -ra -k "cta_pair or staging or not_multiple or fp32_store" > $O/s3y_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s3y_pytest.txt
if grep -q "pytest rc=0" $O/s3y_pytest.txt; then
LIN_AB="0,67108864,2097216,69206080" LIN_SHAPES=igb_large,products timeout 1200 python scripts/bench_linear_shapes.py > $O/s3y_ab.jsonl 2> $O/s3y.err
fi
echo done
