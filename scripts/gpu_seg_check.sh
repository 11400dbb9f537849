#!/bin/bash
# GPU suite (without the 5x5 sweep), C3/C4 bench lines, and the C3 launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider --deselect tests/test_gpu_gaps.py::test_exhaustive_5x5_masks_morphology_and_labelling > gpurun_out/pytest_all.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_all.log
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.log 2>&1
timeout 900 python bench.py --config 4 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.log 2>&1
P3="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-spot-check"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P3 > gpurun_out/ncu_launch.log 2>&1
