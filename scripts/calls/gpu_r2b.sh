#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_advice_r1.py tests/test_gpu_curand_pins.py tests/test_gpu_timed_path.py tests/test_gpu_cast_sweep.py -q -ra --durations=15 > gpurun_out/pytest_new.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_new.txt
echo done
