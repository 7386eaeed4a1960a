#!/bin/bash
# quick HEAD check on one B200: build, the GPU suite, smoke, the default bench line, the reference arm
# usage: scripts/gpu_check.sh <tag>
T=${1:-check}
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${T}_build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -ra --durations=10 > $O/${T}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/${T}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${T}_smoke.txt 2>&1; echo "smoke rc=$?" >> $O/${T}_smoke.txt
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/${T}_bench_ref.json 2>> $O/${T}_bench.err
echo done
