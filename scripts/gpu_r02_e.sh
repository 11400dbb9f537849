#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/tlv.log
VARIANTS="${VARIANTS:-X=0}" bash scripts/gpu_tl_var.sh
P="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
$P > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_launch.log
