#!/bin/bash
# compute-sanitizer over the small sanitizer workload (one tool per run)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --target-processes all \
    python scripts/sanitize_driver.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/sanitize_$tool.log
done
