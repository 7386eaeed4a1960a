#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_propagate.py -q -x > gpurun_out/pytest_prop.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_prop.txt
timeout 600 python scripts/bench_propagate.py > gpurun_out/bench_prop.jsonl 2>&1
PPLOAD_SPMM=scalar timeout 600 python scripts/bench_propagate.py >> gpurun_out/bench_prop.jsonl 2>&1
timeout 1200 python scripts/bench_cpu_oracle.py > gpurun_out/cpu_oracle.jsonl 2> gpurun_out/cpu_oracle.err
tail -2 gpurun_out/pytest_prop.txt; cat gpurun_out/bench_prop.jsonl; wc -l gpurun_out/cpu_oracle.jsonl; tail -2 gpurun_out/cpu_oracle.err
