#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py "tests/test_gpu_parity.py::test_pipelined_graph_calls_match_oracle" "tests/test_gpu_parity.py::test_pipelined_multistream_and_segment_only" -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_pipe.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_pipe.log
rm -f gpurun_out/tlv.log
VARIANTS="${VARIANTS:-X=0}" bash scripts/gpu_tl_var.sh
