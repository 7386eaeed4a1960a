#!/bin/bash
# tests + headline bench + launch list (a shorter round)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -ra > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 3 --skip-e2e --skip-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --steps 20 --warmup 3 --skip-e2e --skip-cpu --skip-k1 --prefetch 0 > gpurun_out/bench_nopf.json 2>> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu --skip-k1 > /dev/null 2>> gpurun_out/ncu.err
echo done
