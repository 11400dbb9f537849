#!/bin/bash
# Parity tests, then A/B of graph replay vs direct launches on the default bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
for v in graph nograph graph; do
  if [ $v = nograph ]; then export FIZI_NO_GRAPH=1; else unset FIZI_NO_GRAPH; fi
  timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1
  echo "bench rc=$?" >> gpurun_out/bench_$v.log
done
unset FIZI_NO_GRAPH
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
