#!/bin/bash
# Round-2 final evidence run (one GPU): full GPU suite, smoke, the driver's
# bench command, every config's bench line, the reference arm, the sharded
# paths on a one-rank group, the checked build + race stress, ncu evidence.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_driver_c3.log 2>&1
bash scripts/gpu_bench_all.sh
timeout 900 python bench.py --steps 300 --warmup 10 > gpurun_out/bench_c3_300.log 2>&1
bash scripts/gpu_sharded.sh
bash scripts/gpu_checks.sh
bash scripts/gpu_profile_r02.sh
