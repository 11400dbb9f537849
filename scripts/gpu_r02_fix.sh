#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider --deselect tests/test_gpu_gaps.py::test_exhaustive_5x5_masks_morphology_and_labelling > gpurun_out/pytest_all.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_all.log
for v in X=0 FIZI_FIX_OLD=1; do
  env $v timeout 600 python bench.py --config 2 --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/fx_c2_$v.log 2>&1
  env $v TL_CONFIG=2 TL_BATCH=64 timeout 300 python scripts/timeline.py > gpurun_out/fx_tl_c2_$v.log 2>&1
done
