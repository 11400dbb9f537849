#!/bin/bash
# the sanitizer substitute: GPU tests + the sanitizer workload on the build
# with device-side invariant checks, then race detection by repetition
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
FIZI_LIB=checked timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/checked_pytest.log 2>&1
echo "pytest (checked build) rc=$?" >> gpurun_out/checked_pytest.log
FIZI_LIB=checked timeout 600 python scripts/sanitize_driver.py > gpurun_out/checked_driver.log 2>&1
echo "driver (checked build) rc=$?" >> gpurun_out/checked_driver.log
timeout 900 python scripts/race_stress.py > gpurun_out/race_stress.log 2>&1
echo "race stress rc=$?" >> gpurun_out/race_stress.log
