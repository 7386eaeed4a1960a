#!/bin/bash
# pairs with one W stage and 10 A slots (experiment bit 33554432): parity, A/B at the row shapes
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3v_build.txt 2>&1
PPLOAD_DEBUG_LINEAR=33554432 timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -x -ra -k "cta_pair or staging or fp32_store or sixteen or f16" > $O/s3v_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s3v_pytest.txt
if grep -q "pytest rc=0" $O/s3v_pytest.txt; then
LIN_AB="0,33554432,2097216,35651648" LIN_SHAPES=igb_large,mag240m timeout 1200 python scripts/bench_linear_shapes.py > $O/s3v_ab.jsonl 2> $O/s3v.err
fi
echo done
