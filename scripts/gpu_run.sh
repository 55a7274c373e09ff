#!/bin/bash
# Generic GPU-box driver: build, then run the commands given as arguments (each a shell string),
# logging to gpurun_out/<tag>.log.  Usage: scripts/gpu_run.sh TAG 'cmd1' 'cmd2' ...
TAG=$1; shift
mkdir -p gpurun_out
exec > >(tee gpurun_out/$TAG.log) 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for c in "$@"; do echo "=== $c"; bash -c "$c"; echo "=== rc=$?"; done
