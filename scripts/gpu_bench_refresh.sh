#!/bin/bash
# refresh the bench lines (final code): driver command, every config, 300-step C3, sharded paths
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_driver_c3.log 2>&1
bash scripts/gpu_bench_all.sh
timeout 900 python bench.py --steps 300 --warmup 10 > gpurun_out/bench_c3_300.log 2>&1
bash scripts/gpu_sharded.sh
