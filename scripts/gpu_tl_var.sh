#!/bin/bash
# timeline variants: VARIANTS = ';'-separated env settings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
i=0
IFS=';' read -ra VS <<< "${VARIANTS:-X=0}"
for v in "${VS[@]}"; do
  for cfgb in "3 64" "5 256"; do
    set -- $cfgb
    echo "=== variant: $v  C$1 B=$2" >> gpurun_out/tlv.log
    eval "env $v TL_CONFIG=$1 TL_BATCH=$2 timeout 300 python scripts/timeline.py" 2>&1 >> gpurun_out/tlv.log
  done
done
