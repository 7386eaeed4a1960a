#!/bin/bash
# Z stored from registers + 2 more A slots (experiment bit 8388608): parity, A/B at products / row shapes
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3n_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -x -ra -k "z_from_registers or not_multiple or cta_pair" > $O/s3n_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s3n_pytest.txt
if grep -q "pytest rc=0" $O/s3n_pytest.txt; then
LIN_AB="0,8388608,2097216,10485824" LIN_SHAPES=products timeout 900 python scripts/bench_linear_shapes.py > $O/s3n_ab.jsonl 2> $O/s3n.err
LIN_AB="0,8388608" LIN_SHAPES=mag240m,igb_large timeout 900 python scripts/bench_linear_shapes.py >> $O/s3n_ab.jsonl 2>> $O/s3n.err
fi
echo done
