#!/bin/bash
# CTA pairs: accumulator-empty arrivals without MEMBAR.ALL.GPU: parity, A/B vs single CTAs, source profile
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s2k_build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_linear_kc.py -q -x -ra > $O/s2k_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s2k_pytest.txt
LIN_AB=0,8192 LIN_SHAPES=mag240m,igb_large timeout 900 python scripts/bench_linear_shapes.py > $O/s2k_ab_pair.jsonl 2> $O/s2k.err
PPLOAD_LINEAR_PAIR=1 LIN_SHAPES=mag240m timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather_linear_kc -s 20 -c 1 -o $O/s2k_pair python scripts/bench_linear_shapes.py > /dev/null 2>> $O/s2k.err
echo done
