#!/bin/bash
# r02 evidence: ncu launch list (C3 bench command) and --set full captures of
# the fused kernels (C3 seg_fast, C5 seg_multi, C4 seg_fast) and the tail
# kernels (C3 morph / ccl / slow words, C4 slow words)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
Q="--no-e2e --no-cpu-baseline --no-spot-check"
P3="python bench.py --steps 3 --warmup 2 $Q"
P5="python bench.py --config 5 --steps 3 --warmup 2 $Q"
P4="python bench.py --config 4 --steps 3 --warmup 2 $Q"
$P3 > gpurun_out/ncu_plain3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P3 > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?" >> gpurun_out/ncu_launch.log
full() {  # name kregex cmd...
  local name=$1 kre=$2; shift 2
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$kre -s 4 -c 1 -f -o gpurun_out/prof_$name "$@" > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?" >> gpurun_out/ncu_$name.log
}
full c3_seg seg_fast $P3
full c3_morph morph_rows $P3
full c3_ccl ccl_kernel $P3
full c3_slow slow_words $P3
$P5 > gpurun_out/ncu_plain5.log 2>&1
full c5_seg seg_multi $P5
$P4 > gpurun_out/ncu_plain4.log 2>&1
full c4_seg seg_fast $P4
full c4_slow slow_words $P4
full c4_ccl ccl_kernel $P4
full c4_morph morph_rows $P4
