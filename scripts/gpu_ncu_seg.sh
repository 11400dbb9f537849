#!/bin/bash
# ncu --set full of one fused segmentation launch (after a plain run of the same command)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${BARGS:-}"
$P > gpurun_out/ncu_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-seg_fast} -s ${KSKIP:-4} -c 1 -o gpurun_out/prof $P > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
./scripts/microbench/stream_bench > gpurun_out/stream.log 2>&1 || true
