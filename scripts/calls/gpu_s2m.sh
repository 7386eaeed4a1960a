#!/bin/bash
# CTA pairs, fp32 TMA path: converted chunks forwarded to the leader by a relay lane; parity + A/B (IGB, MAG)
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s2m_build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_linear_kc.py -q -x -ra > $O/s2m_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s2m_pytest.txt
LIN_AB=0,8192 LIN_SHAPES=igb_large,mag240m timeout 900 python scripts/bench_linear_shapes.py > $O/s2m_ab_pair.jsonl 2> $O/s2m.err
PPLOAD_LINEAR_PAIR=1 LIN_SHAPES=igb_large timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather_linear_kc -s 20 -c 1 -o $O/s2m_pair python scripts/bench_linear_shapes.py > /dev/null 2>> $O/s2m.err
echo done
