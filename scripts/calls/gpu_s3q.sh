#!/bin/bash
# gather4 alone (scripts/micro/gather4_rate.cu): bytes per SM vs box width, stages, issuing warps; LDG reference
O=gpurun_out; mkdir -p $O
(cd scripts/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4_rate gather4_rate.cu -lcuda) > $O/s3q_build.txt 2>&1
timeout 600 ./scripts/micro/gather4_rate > $O/s3q_gather4_rate_lanes.jsonl 2> $O/s3q.err
echo done
