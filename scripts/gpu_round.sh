#!/bin/bash
# one gpurun call: GPU tests, bench lines, ncu launch list + one full capture of the gather
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv > gpurun_out/clocks_start.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -ra > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
for k in 8 299; do
  timeout 300 python bench.py --steps 10 --warmup 3 --per-call $k --skip-e2e --skip-cpu > gpurun_out/bench_k$k.json 2>> gpurun_out/bench.err
done
timeout 300 python bench.py --steps 10 --warmup 3 --chunk 8192 --skip-e2e --skip-cpu > gpurun_out/bench_cr.json 2>> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu > /dev/null 2>> gpurun_out/ncu.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_vec -s 400 -c 2 \
  -o gpurun_out/prof_gather python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu > /dev/null 2>> gpurun_out/ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bucket_rank -s 2 -c 1 \
  -o gpurun_out/prof_rank python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu > /dev/null 2>> gpurun_out/ncu.err
echo done
