#!/bin/bash
# relay arrival with default semantics as the default: all GPU tests, smoke, the three shapes, the bench line
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s42_build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -ra --durations=15 > $O/r2s3f_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/r2s3f_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2s3f_smoke.txt 2>&1; echo "smoke rc=$?" >> $O/r2s3f_smoke.txt
LIN_SHAPES=products,igb_large,mag240m timeout 1200 python scripts/bench_linear_shapes.py > $O/r2s3f_linear_shapes.jsonl 2> $O/r2s3f_linear.err
timeout 1200 python bench.py > $O/r2s3f_bench.json 2> $O/r2s3f_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/r2s3f_bench_ref.json 2>> $O/r2s3f_bench.err
echo done
