#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_dma_spill.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_dma.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_dma.txt
timeout 900 python scripts/bench_configs.py host-cr > gpurun_out/configs_hostcr.jsonl 2> gpurun_out/configs_hostcr.err
rm -f gpurun_out/bench_db2.jsonl; DB_PLACEMENT=host DB_CHUNK=8192 DB_CTAS=8 DB_EPOCHS=2 timeout 900 python scripts/bench_double_buffer.py >> gpurun_out/bench_db2.jsonl 2>> gpurun_out/bench_db2.err
