#!/bin/bash
# closing run of the third session: GPU tests, smoke, the bench line, the reference arm, the ncu launch list
# and a full capture of the headline kernel; A/B of the record pitch (PPLOAD_REC_ALIGN=128: whole L2 lines)
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/s3b_build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -ra --durations=15 > $O/r2s3_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/r2s3_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2s3_smoke.txt 2>&1; echo "smoke rc=$?" >> $O/r2s3_smoke.txt
timeout 1200 python bench.py > $O/r2s3_bench.json 2> $O/r2s3_bench.err
Q="--skip-e2e --skip-cpu --skip-k1 --skip-consumer --skip-double-buffer --skip-next-rows"
rm -f $O/s3b_ab_align.jsonl
for r in 1 2 3; do
  for a in 16 128; do
    PPLOAD_REC_ALIGN=$a timeout 300 python bench.py --steps 30 --warmup 5 $Q 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'rec_align': $a, 'value': d['value'], 'ms_per_step': d['ms_per_step'], 'per_launch_us': d['roofline'].get('per_launch_us'), 'clocks': d['clocks']}))" >> $O/s3b_ab_align.jsonl
  done
done
PPLOAD_REC_ALIGN=128 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_timed_path.py -q -x > $O/s3b_pytest_align128.txt 2>&1; echo "pytest rc=$?" >> $O/s3b_pytest_align128.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/r2s3_bench_ref.json 2>> $O/r2s3_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file $O/r2s3_launches.csv python bench.py --steps 1 --warmup 3 $Q > /dev/null 2>> $O/r2s3_ncu.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_vec -s 60 -c 2 -o $O/r2s3_prof_gather python bench.py --steps 1 --warmup 3 $Q > /dev/null 2>> $O/r2s3_ncu.err
echo done
