#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_storage.py -m gpu -q -ra -x > gpurun_out/pytest_storage.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_storage.txt
df -h /tmp > gpurun_out/storage_probe.txt; mount | grep -E " / | /tmp " >> gpurun_out/storage_probe.txt; lsblk >> gpurun_out/storage_probe.txt 2>&1
rm -f gpurun_out/bench_storage.jsonl
for d in 2 4 8; do PPLOAD_IO_DEPTH=$d timeout 900 python scripts/bench_storage.py >> gpurun_out/bench_storage.jsonl 2>> gpurun_out/bench_storage.err; done
PP_STORAGE_CHUNK=1024 timeout 600 python scripts/bench_storage.py >> gpurun_out/bench_storage.jsonl 2>> gpurun_out/bench_storage.err
