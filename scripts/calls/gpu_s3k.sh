#!/bin/bash
# K-chunked TMA producers: L2 prefetch of the next unit's rows (PPLOAD_LINEAR_PREFETCH=1) A/B; tile mode vs wide
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3k_build.txt 2>&1
PPLOAD_LINEAR_PREFETCH=1 timeout 900 python -m pytest tests/test_gpu_linear_kc.py -q -x -ra > $O/s3k_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s3k_pytest.txt
LIN_AB="0,4194304,E:PPLOAD_LINEAR_PREFETCH=1,E:PPLOAD_LINEAR_PREFETCH=1+PPLOAD_DEBUG_LINEAR=4194304,2097216,E:PPLOAD_LINEAR_PREFETCH=1+PPLOAD_DEBUG_LINEAR=2097216" LIN_SHAPES=products timeout 900 python scripts/bench_linear_shapes.py > $O/s3k_ab.jsonl 2> $O/s3k.err
LIN_AB="0,E:PPLOAD_LINEAR_PREFETCH=1" LIN_SHAPES=mag240m,igb_large timeout 900 python scripts/bench_linear_shapes.py >> $O/s3k_ab.jsonl 2>> $O/s3k.err
echo done
