#!/bin/bash
# K-chunked kernel as the fused-linear default: linear tests (both kernels), products consumer line, A/B
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3d_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_linear.py tests/test_gpu_linear_kc.py -q -x -ra > $O/s3d_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s3d_pytest.txt
LIN_K=8 timeout 900 python scripts/bench_linear.py > $O/s3d_linear_products.jsonl 2> $O/s3d.err
timeout 600 python bench.py --skip-e2e --skip-cpu --skip-k1 --skip-double-buffer --skip-next-rows > $O/s3d_bench_consumer.json 2>> $O/s3d.err
LIN_SHAPES=products timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_linear_kc -s 20 -c 1 -o $O/s3d_prof_kc_products python scripts/bench_linear_shapes.py > /dev/null 2>> $O/s3d.err
echo done
