#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
for v in ${SWEEP_VALUES}; do
  env ${SWEEP_VAR}=$v timeout 600 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_${v}.log 2>&1
  env ${SWEEP_VAR}=$v FIZI_DIAG_NO_FOLD=1 timeout 600 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_${v}_nofold.log 2>&1
done
