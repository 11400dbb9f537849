#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in 64 32 16; do
  FIZI_SUB_FRAMES=$v timeout 300 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_sub$v.log 2>&1
done
