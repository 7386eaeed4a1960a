#!/bin/bash
# CTA pairs as the default of the K-chunked kernel: all fused-linear tests, row-shape and products benches, ncu capture
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s2p_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -x -ra > $O/s2p_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s2p_pytest.txt
timeout 900 python scripts/bench_linear_shapes.py > $O/s2p_linear_shapes.jsonl 2> $O/s2p.err
LIN_K=8 timeout 900 python scripts/bench_linear.py > $O/s2p_linear.jsonl 2>> $O/s2p.err
LIN_SHAPES=mag240m timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_linear_kc -s 20 -c 1 -o $O/s2p_prof_linear_kc python scripts/bench_linear_shapes.py > /dev/null 2>> $O/s2p.err
echo done
