#!/bin/bash
# Full ncu captures of the top kernels of one cfg2 step (run under gpurun, 1 GPU).
# Usage: tools/ncu_full.sh <tag> [workload]
set -u
TAG=${1:-r01}
WL=${2:-cfg2}
OUT=gpurun_out
cap() {  # name regex skip count
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
    --kernel-name-base demangled -k "regex:$2" -s "$3" -c "$4" -o "$OUT/${TAG}_$1" -f \
    python tools/profile_step.py --workload "$WL" > "$OUT/${TAG}_$1.log" 2>&1
  echo "ncu $1 rc=$?"
}
cap modup_inner 'modup_inner' 0 1
cap moddown_tensor 'AddTensor' 0 2
cap rescale 'JobRescale' 0 2
cap modup_passA 'JobModUp' 4 1
cap invgather 'JobInvGather' 0 2
cap decompose 'SrcTensor' 0 2
