#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
python scripts/probe_box.py > gpurun_out/probe.json 2>&1
timeout 900 python -m pytest tests/test_gpu_a2a.py tests/test_gpu_ipc_collective.py tests/test_gpu_ipc.py tests/test_gpu_advice_r1.py tests/test_gpu_exchange.py -q -ra -x > gpurun_out/pytest_r2c.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2c.txt
AVAIL=$(awk '/MemAvailable/ {print int($2/1048576)}' /proc/meminfo)
echo "avail_gb=$AVAIL" >> gpurun_out/probe.json
if [ "$AVAIL" -gt 64 ]; then timeout 600 python scripts/mag240m_dryrun.py > gpurun_out/mag240m.jsonl 2> gpurun_out/mag240m.err; fi
echo done
