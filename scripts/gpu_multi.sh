#!/bin/bash
# exercise the N>1 bench path (torchrun, IPC-linked shards) with 2 ranks on the one GPU
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 5 --warmup 3 --config products > gpurun_out/bench_w2.json 2> gpurun_out/bench_w2.err
echo "rc=$?" >> gpurun_out/bench_w2.err
timeout 600 python -m pytest tests/test_gpu_ipc.py -q > gpurun_out/pytest_ipc.txt 2>&1
echo done
