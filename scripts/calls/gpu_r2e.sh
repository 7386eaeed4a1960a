#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_propagate_sliced.py tests/test_gpu_propagate.py tests/test_gpu_propagate_store.py -q -ra -x > gpurun_out/pytest_r2e.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2e.txt
rm -f gpurun_out/prop.jsonl
for mode in rows sliced; do PPLOAD_SPMM=$mode timeout 600 python scripts/bench_propagate.py >> gpurun_out/prop.jsonl 2>> gpurun_out/prop.err; done

PROP_ONE_HOP=1 PPLOAD_SPMM=sliced timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,sm__inst_executed_pipe_fp64.sum --clock-control none -k regex:"k_spmm|k_slot|k_col" --csv --log-file gpurun_out/ncu_prop_sliced.csv python scripts/bench_propagate.py > /dev/null 2>> gpurun_out/ncu.err
PROP_ONE_HOP=1 PPLOAD_SPMM=sliced timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_sliced -s 5 -c 1 -o gpurun_out/prof_spmm_sliced python scripts/bench_propagate.py > /dev/null 2>> gpurun_out/ncu.err
echo done
