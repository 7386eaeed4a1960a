#!/bin/bash
# fp32 gather4 on a map of (node, hop) rows (K padding = out-of-bounds zero fill): parity, products-shape A/B
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3c_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear_kc.py tests/test_gpu_linear.py -q -x -ra > $O/s3c_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s3c_pytest.txt
LIN_AB="E:PPLOAD_LINEAR=res,E:PPLOAD_LINEAR=kc,E:PPLOAD_LINEAR=kc+PPLOAD_DEBUG_LINEAR=524288,E:PPLOAD_LINEAR=kc+PPLOAD_LINEAR_PAIR=0" LIN_SHAPES=products timeout 900 python scripts/bench_linear_shapes.py > $O/s3c_ab_products.jsonl 2> $O/s3c.err
PPLOAD_LINEAR=kc LIN_SHAPES=products timeout 900 ncu --set full --clock-control none -k regex:k_gather_linear_kc -s 20 -c 1 -o $O/s3c_prof_kc_products python scripts/bench_linear_shapes.py > /dev/null 2>> $O/s3c.err
LIN_SHAPES=products timeout 900 ncu --set full --clock-control none -k regex:"k_gather_linear$" -s 20 -c 1 -o $O/s3c_prof_res_products python scripts/bench_linear_shapes.py > /dev/null 2>> $O/s3c.err
echo done
