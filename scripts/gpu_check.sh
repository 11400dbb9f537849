#!/bin/bash
# One GPU round: parity tests, smoke, a short bench, then ncu (launch list + full capture of the fused kernel).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TESTS=${TESTS:-tests}
timeout 1500 python -m pytest $TESTS -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS:---steps 300 --warmup 10} > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
if [ "${NCU:-1}" = "1" ]; then
  P="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
  $P > gpurun_out/ncu_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_launch.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-seg_fast} -s ${KSKIP:-4} -c 1 -o gpurun_out/prof $P > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_full.log
fi
