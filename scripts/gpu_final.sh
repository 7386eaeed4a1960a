#!/bin/bash
# round-2 closing refresh (second session: after the propagation experiments): GPU tests, smoke, every bench line, secondary configs, (f)-row benches,
# ncu launch list + full captures (with PCIe counters on the host-resident path)
mkdir -p gpurun_out
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/build.txt 2>&1
(cd scripts/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_ceiling hbm_ceiling.cu) >> $O/build.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -ra --durations=20 > $O/r2s2_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/r2s2_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2s2_smoke.txt 2>&1; echo "smoke rc=$?" >> $O/r2s2_smoke.txt
timeout 1200 python bench.py > $O/r2s2_bench.json 2> $O/r2s2_bench.err
timeout 300 python bench.py --chunk 8192 --skip-e2e --skip-cpu --skip-k1 --skip-consumer --skip-double-buffer --skip-next-rows > $O/r2s2_bench_cr.json 2>> $O/r2s2_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/r2s2_bench_ref.json 2>> $O/r2s2_bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --skip-k1 > $O/r2s2_bench_w2_pathcheck.json 2>> $O/r2s2_bench.err
rm -f $O/r2s2_bench_c.jsonl; for k in 1 8; do timeout 120 ./tools/pp_bench_c 20 $k >> $O/r2s2_bench_c.jsonl 2>> $O/r2s2_bench.err; done
timeout 1500 python scripts/bench_configs.py > $O/r2s2_configs.jsonl 2> $O/r2s2_configs.err
LIN_K=8 timeout 900 python scripts/bench_linear.py > $O/r2s2_linear.jsonl 2> $O/r2s2_linear.err
timeout 900 python scripts/bench_linear_shapes.py > $O/r2s2_linear_shapes.jsonl 2>> $O/r2s2_linear.err
timeout 900 python scripts/bench_propagate.py > $O/r2s2_prop.jsonl 2> $O/r2s2_prop.err
timeout 900 python scripts/bench_storage.py > $O/r2s2_storage.jsonl 2> $O/r2s2_storage.err
timeout 900 python scripts/mag240m_dryrun.py > $O/r2s2_mag240m.jsonl 2> $O/r2s2_mag240m.err
Q="--skip-e2e --skip-cpu --skip-k1 --skip-consumer --skip-double-buffer --skip-next-rows"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file $O/r2s2_launches.csv python bench.py --steps 1 --warmup 1 $Q > /dev/null 2>> $O/r2s2_ncu.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_vec -s 60 -c 2 -o $O/r2s2_prof_gather python bench.py --steps 1 --warmup 1 $Q > /dev/null 2>> $O/r2s2_ncu.err
timeout 900 ncu --set full --metrics pcie__read_bytes.sum,pcie__write_bytes.sum --clock-control none --import-source on -k regex:k_gather_tma -s 10 -c 1 -o $O/r2s2_prof_tma_host python bench.py --steps 1 --warmup 3 --skip-cpu --skip-k1 --skip-consumer --skip-double-buffer --skip-next-rows > /dev/null 2>> $O/r2s2_ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bucket_rank|k_scatter|k_hist" -s 3 -c 3 -o $O/r2s2_prof_perm python bench.py --steps 1 --warmup 1 $Q > /dev/null 2>> $O/r2s2_ncu.err
LIN_K=8 LIN_ROUNDS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_gather_linear$" -s 5 -c 1 -o $O/r2s2_prof_linear python scripts/bench_linear.py > /dev/null 2>> $O/r2s2_ncu.err
LIN_SHAPES=mag240m timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_linear_kc -s 20 -c 1 -o $O/r2s2_prof_linear_kc python scripts/bench_linear_shapes.py > /dev/null 2>> $O/r2s2_ncu.err
PROP_ONE_HOP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmm_store_v4 -c 1 -o $O/r2s2_prof_spmm_store python scripts/bench_propagate.py > /dev/null 2>> $O/r2s2_ncu.err
timeout 120 ./scripts/micro/hbm_ceiling > $O/r2s2_hbm_ceiling.jsonl 2>&1
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 $S --tool $tool --num-cuda-barriers 65536 --error-exitcode 9 python -m pytest -q tests/test_gpu_propagate_wave.py \
    -k "not products and not at_scale" > $O/r2s2_sanitize_prop_$tool.txt 2>&1; echo "$tool rc=$?" >> $O/r2s2_sanitize_prop_$tool.txt
done
echo done
