#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/tl_c4.log
for v in ${VARIANTS:-X=0}; do
  echo "=== $v" >> gpurun_out/tl_c4.log
  env $v TL_CONFIG=4 TL_BATCH=64 timeout 300 python scripts/timeline.py >> gpurun_out/tl_c4.log 2>&1
done
