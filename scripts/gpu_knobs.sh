mkdir -p gpurun_out; python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1; rm -f gpurun_out/knobs.jsonl
for cfg in "32 4" "64 4" "32 3" "32 5" "64 3"; do set -- $cfg
  PPLOAD_TILE_ROWS=$1 PPLOAD_GRID_PER_SM=$2 timeout 300 python bench.py --skip-e2e --skip-cpu --skip-consumer --skip-k1 --skip-double-buffer --skip-next-rows 2>/dev/null | sed "s/^{/{\"tile\": $1, \"gps\": $2, /" >> gpurun_out/knobs.jsonl
done
