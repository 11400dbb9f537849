#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_hand.log 2>&1
FIZI_DIAG_NO_FOLD=1 timeout 600 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_nofold.log 2>&1
timeout 600 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline --diag-no-hand > gpurun_out/bench_nohand.log 2>&1
