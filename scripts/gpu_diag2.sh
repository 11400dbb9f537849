#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline --diag-no-masks > gpurun_out/bench_nomask.log 2>&1
timeout 600 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline --diag-no-masks --diag-no-hand > gpurun_out/bench_nomask_nohand.log 2>&1
