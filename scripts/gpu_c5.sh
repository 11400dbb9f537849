#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --config 5 --steps 300 --warmup 10 > gpurun_out/bench_c5.log 2>&1
echo "c5 rc=$?" >> gpurun_out/bench_c5.log
