#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
FIZI_INLINE=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gaps.py tests/test_gpu_pipeline.py -m gpu -q -x --timeout 900 -p no:cacheprovider --deselect tests/test_gpu_gaps.py::test_exhaustive_5x5_masks_morphology_and_labelling > gpurun_out/pytest_inl.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_inl.log
for v in X=0 FIZI_INLINE=1; do
  env $v timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/ab_c3_$v.log 2>&1
  env $v timeout 900 python bench.py --config 4 --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_c4_$v.log 2>&1
done
