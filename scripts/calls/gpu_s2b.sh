#!/bin/bash
# propagation: max L2 fetch granularity experiment (timing + DRAM bytes per hop)
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s2b_build.txt 2>&1
rm -f $O/s2b_prop.jsonl
for g in none 32 64 128 none 32; do
  if [ $g = none ]; then timeout 600 python scripts/bench_propagate.py >> $O/s2b_prop.jsonl 2>> $O/s2b_prop.err
  else PROP_L2FETCH=$g timeout 600 python scripts/bench_propagate.py >> $O/s2b_prop.jsonl 2>> $O/s2b_prop.err; fi
done
for g in none 32; do
  if [ $g = none ]; then E=""; else E="PROP_L2FETCH=$g"; fi
  env $E PROP_ONE_HOP=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --clock-control none -k regex:k_spmm_store_v4 -c 1 --csv python scripts/bench_propagate.py > $O/s2b_ncu_$g.csv 2>> $O/s2b_prop.err
done
echo done
