#!/bin/bash
# one full gpurun call: GPU tests, smoke, bench lines, secondary configs, (f)-row benches, ncu launch list + full captures
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -ra > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --chunk 8192 --skip-e2e --skip-cpu --skip-k1 --skip-consumer --skip-double-buffer --skip-next-rows > gpurun_out/bench_cr.json 2>> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
rm -f gpurun_out/bench_c.jsonl; for k in 1 8; do timeout 120 ./tools/pp_bench_c 20 $k >> gpurun_out/bench_c.jsonl 2>> gpurun_out/bench.err; done
timeout 1500 python scripts/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
rm -f gpurun_out/bench_linear.jsonl; for k in 1 8 299; do LIN_K=$k timeout 600 python scripts/bench_linear.py >> gpurun_out/bench_linear.jsonl 2>> gpurun_out/bench_linear.err; done
timeout 600 python scripts/bench_propagate.py > gpurun_out/bench_prop.jsonl 2> gpurun_out/bench_prop.err
timeout 900 python scripts/bench_storage.py > gpurun_out/bench_storage.jsonl 2> gpurun_out/bench_storage.err
timeout 900 python scripts/bench_configs.py papers100M-labelled host-cr > gpurun_out/configs2.jsonl 2>> gpurun_out/configs.err
rm -f gpurun_out/bench_db.jsonl; for pl in hbm host; do DB_PLACEMENT=$pl DB_CHUNK=8192 DB_CTAS=8 DB_EPOCHS=2 timeout 900 python scripts/bench_double_buffer.py >> gpurun_out/bench_db.jsonl 2>> gpurun_out/bench_db.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu --skip-k1 --skip-consumer --skip-double-buffer --skip-next-rows > /dev/null 2>> gpurun_out/ncu.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_vec -s 60 -c 2 \
  -o gpurun_out/prof_gather python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu --skip-k1 --skip-consumer --skip-double-buffer --skip-next-rows > /dev/null 2>> gpurun_out/ncu.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_tma -s 10 -c 1 \
  -o gpurun_out/prof_tma_spill python bench.py --steps 1 --warmup 1 --skip-cpu --skip-k1 --skip-consumer --skip-double-buffer --skip-next-rows > /dev/null 2>> gpurun_out/ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bucket_rank|k_scatter|k_hist" -s 3 -c 3 \
  -o gpurun_out/prof_perm python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu --skip-k1 --skip-consumer --skip-double-buffer --skip-next-rows > /dev/null 2>> gpurun_out/ncu.err
LIN_K=8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather_linear -s 5 -c 1 \
  -o gpurun_out/prof_linear python scripts/bench_linear.py > /dev/null 2>> gpurun_out/ncu.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_store_v4 -s 1 -c 1 \
  -o gpurun_out/prof_spmm_store python scripts/bench_propagate.py > /dev/null 2>> gpurun_out/ncu.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assemble_staged -s 40 -c 1 \
  -o gpurun_out/prof_assemble python scripts/bench_storage.py > /dev/null 2>> gpurun_out/ncu.err
echo done
