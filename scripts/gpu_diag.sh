#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline --diag-no-hand > gpurun_out/bench_nohand.log 2>&1
timeout 600 python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_hand.log 2>&1
P="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
$P > gpurun_out/ncu_plain.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-seg_fast}" -s ${KSKIP:-4} -c ${KCOUNT:-1} -o gpurun_out/prof $P > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full.log
