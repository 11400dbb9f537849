#!/bin/bash
# round 2: all GPU tests + smoke + C3/C5/C4 bench lines (no ncu)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
echo "c3 rc=$?" >> gpurun_out/bench_c3.log
timeout 600 python bench.py --config 5 --steps 300 --warmup 10 > gpurun_out/bench_c5.log 2>&1
echo "c5 rc=$?" >> gpurun_out/bench_c5.log
timeout 600 python bench.py --config 4 --steps 40 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
echo "c4 rc=$?" >> gpurun_out/bench_c4.log
