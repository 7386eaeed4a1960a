#!/bin/bash
# cp.async-staged row kernel for propagation: parity, timing vs the register row kernel, ncu DRAM
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s2d_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_propagate_wave.py -q -x -ra > $O/s2d_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s2d_pytest.txt
rm -f $O/s2d_prop.jsonl
run() { env "$@" timeout 600 python scripts/bench_propagate.py | sed "s/^/{\"env\": \"$*\", \"r\": /; s/$/}/" >> $O/s2d_prop.jsonl 2>> $O/s2d_prop.err; }
run PPLOAD_SPMM=rows
for v in 0 1 2 3; do run PPLOAD_SPMM=cp PPLOAD_CP_VARIANT=$v; done
run PPLOAD_SPMM=rows
run PPLOAD_SPMM=cp
for v in rows cp; do
  PPLOAD_SPMM=$v PROP_ONE_HOP=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_spmm" -c 1 --csv python scripts/bench_propagate.py > $O/s2d_ncu_$v.csv 2>> $O/s2d_prop.err
done
echo done
