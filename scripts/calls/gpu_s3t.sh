#!/bin/bash
# 512-byte gather4 boxes for chunk pairs at any even chunk count (PPLOAD_LINEAR_TMA_F32=3): parity, IGB-large / products A/B
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3t_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -x -ra -k "whole_tile or not_multiple or staging or cta_pair" > $O/s3t_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s3t_pytest.txt
if grep -q "pytest rc=0" $O/s3t_pytest.txt; then
LIN_AB="0,E:PPLOAD_LINEAR_TMA_F32=3,2097216,E:PPLOAD_LINEAR_TMA_F32=3+PPLOAD_DEBUG_LINEAR=2097216" LIN_SHAPES=igb_large,products timeout 1200 python scripts/bench_linear_shapes.py > $O/s3t_ab.jsonl 2> $O/s3t.err
fi
echo done
