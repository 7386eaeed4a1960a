#!/bin/bash
# CTA pairs: W stages 2 / 3 / 4 (A slots 8 / 6 / 4) vs single CTAs at IGB and MAG rows
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s2o_build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -x -ra > $O/s2o_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s2o_pytest.txt
LIN_AB=0,8192,139264,73728 LIN_SHAPES=igb_large,mag240m timeout 1200 python scripts/bench_linear_shapes.py > $O/s2o_ab_pair.jsonl 2> $O/s2o.err
echo done
