#!/bin/bash
# bench lines of every config at N = 1 (default args = the driver's C3 line)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
timeout 600 python bench.py --config 2 --steps 300 --warmup 10 > gpurun_out/bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c2.log
timeout 600 python bench.py --config 5 --steps 300 --warmup 10 > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
timeout 900 python bench.py --config 4 --steps 40 --warmup 5 > gpurun_out/bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4.log
timeout 300 python bench.py --config 1 --steps 300 --warmup 10 > gpurun_out/bench_c1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c1.log
