#!/bin/bash
# final run of round 2: GPU tests, smoke, the full bench line, the reference arm, ncu launch list of the bench
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3u_build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -ra --durations=15 > $O/r2s3d_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/r2s3d_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2s3d_smoke.txt 2>&1; echo "smoke rc=$?" >> $O/r2s3d_smoke.txt
timeout 1200 python bench.py > $O/r2s3d_bench.json 2> $O/r2s3d_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/r2s3d_bench_ref.json 2>> $O/r2s3d_bench.err
echo done
