#!/bin/bash
# epilogue: next slice's TMEM loads split around the staging stores (bit 134217728: old order): parity, A/B
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s41_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -x -ra > $O/s41_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s41_pytest.txt
if grep -q "pytest rc=0" $O/s41_pytest.txt; then
LIN_AB="0,134217728" LIN_SHAPES=products,igb_large,mag240m timeout 1200 python scripts/bench_linear_shapes.py > $O/s41_ab.jsonl 2> $O/s41.err
fi
echo done
