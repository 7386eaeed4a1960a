#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "event_double or double_buffer or tiny_epoch" > gpurun_out/pytest_db.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_db.txt
timeout 900 python scripts/bench_double_buffer.py > gpurun_out/bench_db.jsonl 2> gpurun_out/bench_db.err
