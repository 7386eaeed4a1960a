#!/bin/bash
# exchange-copy parity (loopback + 2-process IPC) and the W=2 bench path on the one GPU
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_exchange.py tests/test_gpu_ipc.py -q -x -ra > gpurun_out/pytest_exchange.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_exchange.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "loopback or gather_paths" > gpurun_out/pytest_loopback.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_loopback.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 5 --warmup 3 --config products --skip-e2e --skip-consumer --skip-double-buffer --skip-next-rows > gpurun_out/bench_w2.json 2> gpurun_out/bench_w2.err
echo "rc=$?" >> gpurun_out/bench_w2.err
tail -3 gpurun_out/pytest_exchange.txt gpurun_out/pytest_loopback.txt; tail -c 1500 gpurun_out/bench_w2.json; tail -2 gpurun_out/bench_w2.err
