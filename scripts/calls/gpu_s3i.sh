#!/bin/bash
# closing run after the fused-linear default change: GPU tests, smoke, the full bench line, the reference arm
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3i_build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -ra --durations=15 > $O/r2s3b_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/r2s3b_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2s3b_smoke.txt 2>&1; echo "smoke rc=$?" >> $O/r2s3b_smoke.txt
timeout 1200 python bench.py > $O/r2s3b_bench.json 2> $O/r2s3b_bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --skip-k1 > $O/r2s3b_bench_w2_pathcheck.json 2>> $O/r2s3b_bench.err
echo done
