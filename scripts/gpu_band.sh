#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_b16.log 2>&1
cp paper_1907_04393_b200/libfizi.so /tmp/keep.so; cp paper_1907_04393_b200/libfizi_b8.so paper_1907_04393_b200/libfizi.so
timeout 300 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_b8.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "config or exhaustive or random_32" -p no:cacheprovider > gpurun_out/pytest_b8.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_b8.log
cp /tmp/keep.so paper_1907_04393_b200/libfizi.so
