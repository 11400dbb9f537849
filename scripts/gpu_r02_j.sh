#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_pipe.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_pipe.log
bash scripts/gpu_r02_h.sh
