#!/bin/bash
# A/B of an alternative build (ALT=path of a .so) against the in-tree libfizi.so on the timeline
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
: > gpurun_out/ab_lib.log
for r in 1 2; do
  echo "=== default" >> gpurun_out/ab_lib.log
  timeout 300 python scripts/timeline.py 2>&1 | tail -1 >> gpurun_out/ab_lib.log
  cp paper_1907_04393_b200/libfizi.so /tmp/libfizi_keep.so
  cp $ALT paper_1907_04393_b200/libfizi.so
  echo "=== $ALT" >> gpurun_out/ab_lib.log
  timeout 300 python scripts/timeline.py 2>&1 | tail -1 >> gpurun_out/ab_lib.log
  cp /tmp/libfizi_keep.so paper_1907_04393_b200/libfizi.so
done
