#!/bin/bash
# CTA pairs with 2 W stages + 8 A slots: parity; A/B single / pair (new layout) / pair (old layout) at IGB and MAG rows
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s2n_build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -x -ra > $O/s2n_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s2n_pytest.txt
LIN_AB=0,8192,73728 LIN_SHAPES=igb_large,mag240m timeout 1200 python scripts/bench_linear_shapes.py > $O/s2n_ab_pair.jsonl 2> $O/s2n.err
echo done
