#!/bin/bash
# order[] entries one unit ahead in the K-chunked TMA producers: parity, A/B at products / MAG240M / IGB-large rows
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3f_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -x -ra > $O/s3f_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s3f_pytest.txt
LIN_AB="0,1048576,66,1048642" LIN_SHAPES=products timeout 900 python scripts/bench_linear_shapes.py > $O/s3f_ab.jsonl 2> $O/s3f.err
LIN_AB="0,1048576" LIN_SHAPES=mag240m,igb_large timeout 900 python scripts/bench_linear_shapes.py >> $O/s3f_ab.jsonl 2>> $O/s3f.err
echo done
