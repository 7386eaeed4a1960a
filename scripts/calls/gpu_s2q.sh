#!/bin/bash
# (tile, hop) work units over the whole grid (pairs: 74 instead of 72): parity, A/B on vs off (bit 262144)
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s2q_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -x -ra > $O/s2q_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s2q_pytest.txt
if grep -q "pytest rc=0" $O/s2q_pytest.txt; then
  LIN_AB=0,262144 LIN_SHAPES=mag240m,igb_large timeout 1200 python scripts/bench_linear_shapes.py > $O/s2q_ab_units.jsonl 2> $O/s2q.err
fi
echo done
