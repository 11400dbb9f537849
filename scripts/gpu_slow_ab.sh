#!/bin/bash
# C4: per-pixel word kernel, ALU test (default) vs colour-table build; ncu of the default one
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
: > gpurun_out/slow_ab.log
P="python bench.py --config 4 --steps 40 --warmup 5 --no-e2e --no-cpu-baseline"
for r in 1 2; do
  echo "=== alu" >> gpurun_out/slow_ab.log
  timeout 600 $P 2>&1 | tail -1 | cut -c1-200 >> gpurun_out/slow_ab.log
  timeout 600 $P 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['stage_ms_per_step'])" >> gpurun_out/slow_ab.log 2>&1
  cp paper_1907_04393_b200/libfizi.so /tmp/libfizi_keep.so
  cp paper_1907_04393_b200/libfizi_table.so paper_1907_04393_b200/libfizi.so
  echo "=== table" >> gpurun_out/slow_ab.log
  timeout 600 $P 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['stage_ms_per_step'])" >> gpurun_out/slow_ab.log 2>&1
  cp /tmp/libfizi_keep.so paper_1907_04393_b200/libfizi.so
done
Q="python bench.py --config 4 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:slow_words -s 2 -c 1 -o gpurun_out/prof_slow $Q > gpurun_out/ncu_slow.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_slow.log
