#!/bin/bash
# wave-synchronous propagation: parity, timing sweep vs the row kernels, ncu DRAM bytes per hop
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s2c_build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_propagate_wave.py tests/test_gpu_propagate.py tests/test_gpu_propagate_store.py -q -x -ra > $O/s2c_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/s2c_pytest.txt
rm -f $O/s2c_prop.jsonl
run() { env "$@" timeout 600 python scripts/bench_propagate.py | sed "s/^/{\"env\": \"$*\", \"r\": /; s/$/}/" >> $O/s2c_prop.jsonl 2>> $O/s2c_prop.err; }
run PPLOAD_SPMM=rows
run PPLOAD_SPMM=wave
run PPLOAD_SPMM=wave PPLOAD_WAVE_VARIANT=1
run PPLOAD_SPMM=wave PPLOAD_WAVE_VARIANT=2
run PPLOAD_SPMM=wave PPLOAD_WAVE_WINDOWS=16
run PPLOAD_SPMM=wave PPLOAD_WAVE_WINDOWS=64
run PPLOAD_SPMM=wave PPLOAD_WAVE_LAG=0
run PPLOAD_SPMM=wave PPLOAD_WAVE_LAG=1
run PPLOAD_SPMM=wave PPLOAD_WAVE_LAG=4
for v in rows wave; do
  PPLOAD_SPMM=$v PROP_ONE_HOP=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_spmm" -c 1 --csv python scripts/bench_propagate.py > $O/s2c_ncu_$v.csv 2>> $O/s2c_prop.err
done
echo done
