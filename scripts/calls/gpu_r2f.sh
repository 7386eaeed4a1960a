#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
PPLOAD_SPMM_WINDOW=16 timeout 900 python -m pytest tests/test_gpu_propagate_sliced.py -q -x > gpurun_out/pytest_r2f.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2f.txt
PPLOAD_SPMM_WINDOW=16 PPLOAD_SPMM=sliced timeout 600 python scripts/bench_propagate.py > gpurun_out/prop16.jsonl 2>> gpurun_out/prop.err
PROP_ONE_HOP=1 PPLOAD_SPMM_WINDOW=16 PPLOAD_SPMM=sliced timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,lts__t_sectors_srcunit_tex_evict_last_lookup_hit.sum,lts__t_sectors_srcunit_tex_evict_last_lookup_miss.sum,lts__t_requests_srcunit_ltcfabric.sum --clock-control none -k regex:"k_spmm" --csv --log-file gpurun_out/ncu_prop16.csv python scripts/bench_propagate.py > /dev/null 2>> gpurun_out/ncu.err
