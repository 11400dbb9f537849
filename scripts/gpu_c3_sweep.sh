#!/bin/bash
# C3 bench under launch-parameter switches (VARS = space-separated ENV=VAL)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in ${VARS:-X=0}; do
  env $v timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/sw_c3_$v.log 2>&1
done
