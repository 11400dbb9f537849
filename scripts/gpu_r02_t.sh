#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_parity.py -k "pipelined or pipeline or track_runs or reset" -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_t.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_t.log
rm -f gpurun_out/tlv.log
VARIANTS="${VARIANTS:-X=0}" bash scripts/gpu_tl_var.sh
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.log 2>&1
timeout 600 python bench.py --config 5 --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.log 2>&1
