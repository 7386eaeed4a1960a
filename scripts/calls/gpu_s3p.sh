#!/bin/bash
# hybrid A side (bit 16777216): chunk 1 by LDG in the gather warps; parity, products A/B
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3p_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -x -ra -k "hybrid or not_multiple or cta_pair" > $O/s3p_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s3p_pytest.txt
if grep -q "pytest rc=0" $O/s3p_pytest.txt; then
LIN_AB="0,16777216,2097216,18874432,E:PPLOAD_LINEAR_PAIR=0+PPLOAD_DEBUG_LINEAR=16777216" LIN_SHAPES=products timeout 900 python scripts/bench_linear_shapes.py > $O/s3p_ab.jsonl 2> $O/s3p.err
fi
echo done
