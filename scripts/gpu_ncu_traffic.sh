#!/bin/bash
# Per-kernel DRAM traffic of a few pipelined calls (after a plain run of the same command)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/timeline.py > gpurun_out/ncu_tr_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv \
  -s 200 -c 40 --log-file gpurun_out/traffic.csv python scripts/timeline.py > gpurun_out/ncu_tr.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_tr.log
