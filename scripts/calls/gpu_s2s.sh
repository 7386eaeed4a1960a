#!/bin/bash
# fp32 records by wide (256-B, unswizzled) gather4 boxes: parity, interleaved A/B vs 128-B halves at IGB-large rows
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s2s_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -x -ra > $O/s2s_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s2s_pytest.txt
if grep -q "pytest rc=0" $O/s2s_pytest.txt; then
  LIN_AB="0,E:PPLOAD_LINEAR_TMA_F32=2,E:PPLOAD_LINEAR_PAIR=0,E:PPLOAD_LINEAR_PAIR=0+PPLOAD_LINEAR_TMA_F32=2" LIN_SHAPES=igb_large timeout 1200 python scripts/bench_linear_shapes.py > $O/s2s_ab_wide.jsonl 2> $O/s2s.err
fi
echo done
