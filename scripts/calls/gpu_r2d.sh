#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_ipc_collective.py -q -ra -x > gpurun_out/pytest_r2d.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2d.txt
timeout 900 python bench.py --steps 20 --warmup 3 --skip-double-buffer --skip-next-rows > gpurun_out/bench1.json 2> gpurun_out/bench1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
echo done
