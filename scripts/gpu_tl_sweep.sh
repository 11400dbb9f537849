#!/bin/bash
# timeline.py under a set of env variants (SWEEP = ';'-separated env strings)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/tl_sweep.log
IFS=';' read -ra VS <<< "${SWEEP:-}"
for v in "${VS[@]}"; do
  echo "=== $v" >> gpurun_out/tl_sweep.log
  eval "env $v timeout 300 python scripts/timeline.py" 2>&1 | tail -1 >> gpurun_out/tl_sweep.log
done
