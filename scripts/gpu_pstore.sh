#!/bin/bash
# store propagation: parity tests + bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_propagate_store.py tests/test_gpu_propagate.py -m gpu -q -ra -x > gpurun_out/pytest_pstore.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pstore.txt
timeout 600 python scripts/bench_propagate.py > gpurun_out/bench_prop.jsonl 2> gpurun_out/bench_prop.err
