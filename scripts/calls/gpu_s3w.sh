#!/bin/bash
# issuing lanes at the row shapes, whole kernel and A side alone (bit 2097216), one process per shape
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3w_build.txt 2>&1
PPLOAD_LINEAR_ISSUE_LANES=4 timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -x -ra -k "cta_pair or staging or not_multiple" > $O/s3w_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s3w_pytest.txt
if grep -q "pytest rc=0" $O/s3w_pytest.txt; then
LIN_AB="E:PPLOAD_LINEAR_ISSUE_LANES=1,E:PPLOAD_LINEAR_ISSUE_LANES=4,E:PPLOAD_LINEAR_ISSUE_LANES=1+PPLOAD_DEBUG_LINEAR=2097216,E:PPLOAD_LINEAR_ISSUE_LANES=4+PPLOAD_DEBUG_LINEAR=2097216" LIN_SHAPES=igb_large,mag240m timeout 1500 python scripts/bench_linear_shapes.py > $O/s3w_ab.jsonl 2> $O/s3w.err
fi
echo done
