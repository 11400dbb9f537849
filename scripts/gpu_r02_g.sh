#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_parity.py -k "config5 or multistream or pipelined" -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_c5.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_c5.log
for v in ${C5VARS:-X=0}; do
  env $v timeout 600 python bench.py --config 5 --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c5_$v.log 2>&1
done
