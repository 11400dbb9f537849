#!/bin/bash
# Build locally (incremental), then run a command on the GPU box via gpurun.
# usage: scripts/grun.sh TIMEOUT 'command'
cd /root/repo
python -c "import __graft_entry__ as g; from paper_1907_04393_b200 import build as b; b.build(); b.build_checked(); import synth; synth.build_dev()" || exit 9
exec /usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
