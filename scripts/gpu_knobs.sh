#!/bin/bash
# headline sensitivity to the prefetched permutation's CTA cap
mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1; rm -f gpurun_out/knobs.jsonl
for rep in 1 2; do for c in 148 296 444; do
  PPLOAD_PREFETCH_CTAS=$c timeout 300 python bench.py --skip-e2e --skip-cpu --skip-consumer --skip-k1 --skip-double-buffer --skip-next-rows 2>/dev/null | sed "s/^{/{\"prefetch_ctas\": $c, /" >> gpurun_out/knobs.jsonl
done; done
