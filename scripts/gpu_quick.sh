#!/bin/bash
# Quick bench variants (no e2e / cpu baseline).  VARIANTS = ';'-separated
# "ENV=.. ENV2=..|extra bench args" entries; q_0 is the default run.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 300 > gpurun_out/q_0.log 2>&1
i=0
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for v in "${VS[@]}"; do
  i=$((i+1))
  envs="${v%%|*}"; args="${v#*|}"
  eval "env $envs timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 300 $args" > gpurun_out/q_$i.log 2>&1
  echo "variant: $v" >> gpurun_out/q_$i.log
done
