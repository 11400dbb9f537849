#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider --deselect tests/test_gpu_gaps.py::test_exhaustive_5x5_masks_morphology_and_labelling > gpurun_out/pytest_all.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_all.log
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.log 2>&1
timeout 600 python bench.py --force-gather --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_fg.log 2>&1
timeout 600 python bench.py --config 5 --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
