#!/bin/bash
# synccheck over the propagation kernels with room for the bulk-copy variants' mbarriers (32 warps x 12 per CTA)
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s2g_build.txt 2>&1
S=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $S --tool synccheck --num-cuda-barriers 65536 --error-exitcode 9 python -m pytest -q tests/test_gpu_propagate_wave.py \
  -k "not products and not at_scale" > $O/s2g_synccheck.txt 2>&1; echo "synccheck rc=$?" >> $O/s2g_synccheck.txt
echo done
