#!/bin/bash
# (1) propagation bulk-copy variant 7 (256 x 48 slots; rerun after the 64-bit parity-mask fix); (2) fused linear: Z-write wait at exit, A/B
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s2f_build.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_propagate_wave.py -q -x -ra -k cp > $O/s2f_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s2f_pytest.txt
timeout 600 python -m pytest tests/test_gpu_linear.py tests/test_gpu_linear_kc.py -q -x -ra > $O/s2f_pytest_linear.txt 2>&1; echo "pytest rc=$?" >> $O/s2f_pytest_linear.txt
rm -f $O/s2f_prop.jsonl
run() { env "$@" timeout 240 python scripts/bench_propagate.py | sed "s/^/{\"env\": \"$*\", \"r\": /; s/$/}/" >> $O/s2f_prop.jsonl 2>> $O/s2f_prop.err; }
if grep -q "pytest rc=0" $O/s2f_pytest.txt; then
  run PPLOAD_SPMM=cp PPLOAD_CP_VARIANT=7
fi
LIN_AB=0,131072 LIN_SHAPES=products,mag240m,igb_large timeout 1200 python scripts/bench_linear_shapes.py > $O/s2f_linear_ab.jsonl 2> $O/s2f_linear.err
echo done
