#!/bin/bash
# Secondary bench lines: C4 (3840x2160, one stream) and C5 (256 streams of
# 640x480, per-stream envelopes), N = 1.  The default bench line is C3.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --config 4 --steps 40 --warmup 5 > gpurun_out/bench_c4.log 2>&1
echo "c4 rc=$?" >> gpurun_out/bench_c4.log
timeout 900 python bench.py --config 5 --steps 300 --warmup 10 > gpurun_out/bench_c5.log 2>&1
echo "c5 rc=$?" >> gpurun_out/bench_c5.log
