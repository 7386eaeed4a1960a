#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_storage.py -m gpu -q -ra -x > gpurun_out/pytest_storage.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_storage.txt
rm -f gpurun_out/bench_storage.jsonl
for io in posix; do PPLOAD_IO=$io timeout 900 python scripts/bench_storage.py 2>> gpurun_out/bench_storage.err | sed "s/^{/{\"io\": \"$io\", /" >> gpurun_out/bench_storage.jsonl; done
