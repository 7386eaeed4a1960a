#!/bin/bash
# wide fp32 gather4 as the default: K-chunked parity, products-shape A/B (resident kernel vs K-chunked
# with halves / wide boxes, pairs / single), IGB-large rows at the new default
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3a_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -x -ra > $O/s3a_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s3a_pytest.txt
LIN_AB="E:PPLOAD_LINEAR=res,E:PPLOAD_LINEAR=kc,E:PPLOAD_LINEAR=kc+PPLOAD_LINEAR_TMA_F32=1,E:PPLOAD_LINEAR=kc+PPLOAD_LINEAR_PAIR=0" LIN_SHAPES=products timeout 900 python scripts/bench_linear_shapes.py > $O/s3a_ab_products.jsonl 2> $O/s3a.err
LIN_SHAPES=igb_large,mag240m timeout 900 python scripts/bench_linear_shapes.py > $O/s3a_shapes.jsonl 2>> $O/s3a.err
echo done
