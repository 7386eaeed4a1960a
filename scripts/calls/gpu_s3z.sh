#!/bin/bash
# relay arrival with default semantics as the default: all GPU tests, smoke, the three shapes, the bench line
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3z_build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -ra --durations=15 > $O/r2s3e_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/r2s3e_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2s3e_smoke.txt 2>&1; echo "smoke rc=$?" >> $O/r2s3e_smoke.txt
LIN_AB="0,67108864" LIN_SHAPES=products,igb_large,mag240m timeout 1200 python scripts/bench_linear_shapes.py > $O/r2s3e_linear_shapes.jsonl 2> $O/r2s3e_linear.err
timeout 1200 python bench.py > $O/r2s3e_bench.json 2> $O/r2s3e_bench.err
echo done
