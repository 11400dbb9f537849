#!/bin/bash
mkdir -p gpurun_out
TL_CONFIG=4 TL_WARM=3 TL_NCALLS=10 timeout 300 python scripts/timeline.py > gpurun_out/tl_c4.log 2>&1
TL_CONFIG=2 TL_WARM=3 TL_NCALLS=12 timeout 300 python scripts/timeline.py > gpurun_out/tl_c2.log 2>&1
