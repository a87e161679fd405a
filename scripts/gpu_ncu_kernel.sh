#!/bin/bash
# One ncu --set full capture (source-level) of a named kernel during a short bench leg.
#   scripts/gpu_ncu_kernel.sh <kernel-regex> <workloads> <out-name> [launch-skip]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K=$1; WL=$2; OUT=$3; SKIP=${4:-6}
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$K" -s $SKIP -c 1 \
  -o gpurun_out/$OUT -f python bench.py --workloads $WL --steps 3 --warmup 3 --cpu-seconds 0.2 > gpurun_out/$OUT.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/$OUT.log
