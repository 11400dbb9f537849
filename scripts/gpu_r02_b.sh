#!/bin/bash
# round 2: new parity tests + C2 full sequence + timelines (host cost per call)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gaps.py tests/test_relearn.py "tests/test_gpu_parity.py::test_config2_lighting_drift_full_sequence" tests/test_gpu_parity.py::test_device_generator_matches_host -m gpu -q --timeout 1200 -p no:cacheprovider --durations=10 > gpurun_out/pytest_gaps.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gaps.log
timeout 300 python scripts/timeline.py > gpurun_out/tl_c3.log 2>&1
TL_CONFIG=5 TL_BATCH=256 timeout 300 python scripts/timeline.py > gpurun_out/tl_c5.log 2>&1
