mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -ra -x > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
nvidia-smi -q | grep -iE "product name|pcie|link gen|width|bus id" | head -20 > gpurun_out/probe.txt; nproc >> gpurun_out/probe.txt; free -g >> gpurun_out/probe.txt
