#!/bin/bash
# propagation: one cp.async.bulk per neighbour row (variants 4-7) vs the register row kernel
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s2e_build.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_propagate_wave.py -q -x -ra -k cp > $O/s2e_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s2e_pytest.txt
rm -f $O/s2e_prop.jsonl
run() { env "$@" timeout 240 python scripts/bench_propagate.py | sed "s/^/{\"env\": \"$*\", \"r\": /; s/$/}/" >> $O/s2e_prop.jsonl 2>> $O/s2e_prop.err; }
run PPLOAD_SPMM=rows
for v in 4 5 6 7; do run PPLOAD_SPMM=cp PPLOAD_CP_VARIANT=$v; done
run PPLOAD_SPMM=rows
for v in rows cp; do
  PPLOAD_CP_VARIANT=4 PPLOAD_SPMM=$v PROP_ONE_HOP=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_requests_srcunit_tex_op_read.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"k_spmm" -c 1 --csv python scripts/bench_propagate.py > $O/s2e_ncu_$v.csv 2>> $O/s2e_prop.err
done
echo done
