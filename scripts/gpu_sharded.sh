#!/bin/bash
# the sharded paths on a one-rank NCCL group (--force-gather): C3 and C5
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --force-gather --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_fg.log 2>&1
echo "rc=$?" >> gpurun_out/bench_c3_fg.log
timeout 600 python bench.py --config 5 --force-gather --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_fg.log 2>&1
echo "rc=$?" >> gpurun_out/bench_c5_fg.log
