#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider --deselect tests/test_gpu_gaps.py::test_exhaustive_5x5_masks_morphology_and_labelling > gpurun_out/pytest_all.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_all.log
rm -f gpurun_out/tlv.log
VARIANTS="${VARIANTS:-X=0}" bash scripts/gpu_tl_var.sh
