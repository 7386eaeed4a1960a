#!/bin/bash
# gather4 issued from several lanes per gather warp (PPLOAD_LINEAR_ISSUE_LANES): parity, A/B at the three shapes
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3r_build.txt 2>&1
PPLOAD_LINEAR_ISSUE_LANES=4 timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -x -ra > $O/s3r_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s3r_pytest.txt
if grep -q "pytest rc=0" $O/s3r_pytest.txt; then
L="E:PPLOAD_LINEAR_ISSUE_LANES=1,E:PPLOAD_LINEAR_ISSUE_LANES=2,E:PPLOAD_LINEAR_ISSUE_LANES=4,E:PPLOAD_LINEAR_ISSUE_LANES=8"
LIN_AB="$L,E:PPLOAD_LINEAR_ISSUE_LANES=1+PPLOAD_DEBUG_LINEAR=2097216,E:PPLOAD_LINEAR_ISSUE_LANES=4+PPLOAD_DEBUG_LINEAR=2097216" LIN_SHAPES=products timeout 900 python scripts/bench_linear_shapes.py > $O/s3r_ab.jsonl 2> $O/s3r.err
LIN_AB="$L" LIN_SHAPES=mag240m,igb_large timeout 900 python scripts/bench_linear_shapes.py >> $O/s3r_ab.jsonl 2>> $O/s3r.err
fi
echo done
