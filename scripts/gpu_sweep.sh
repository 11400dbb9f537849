#!/bin/bash
# parity tests + bench sweep over an env var (SWEEP_VAR / SWEEP_VALUES)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
for v in ${SWEEP_VALUES:-16}; do
  env ${SWEEP_VAR:-FIZI_SUB_FRAMES}=$v timeout 600 python bench.py ${BENCH_ARGS:---steps 300 --warmup 10 --no-e2e --no-cpu-baseline} > gpurun_out/bench_${v}.log 2>&1
done
