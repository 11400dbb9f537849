#!/bin/bash
# C4 launch-parameter sweep (labelling threads, morphology warps per CTA)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
: > gpurun_out/c4_sweep.log
P="python bench.py --config 4 --steps 40 --warmup 5 --no-e2e --no-cpu-baseline"
for v in "X=0" "FIZI_CCL_THREADS=1024" "FIZI_CCL_THREADS=256" "FIZI_MORPH_WARPS=2" "FIZI_MORPH_WARPS=8" "X=0"; do
  echo "=== $v" >> gpurun_out/c4_sweep.log
  env $v timeout 600 $P 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['value']), {k: round(v*1e3,1) for k,v in d['roofline']['stage_ms_per_step'].items()})" >> gpurun_out/c4_sweep.log 2>&1
done
