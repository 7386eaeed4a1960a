#!/bin/bash
# fused-linear suites after making whole-tile boxes / TMA-path L2 prefetch opt-in
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3l_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -x -ra > $O/s3l_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s3l_pytest.txt
LIN_SHAPES=products,igb_large,mag240m timeout 900 python scripts/bench_linear_shapes.py > $O/s3l_shapes.jsonl 2> $O/s3l.err
echo done
