#!/bin/bash
# Full ncu captures of the top kernels of one step (run under gpurun, 1 GPU).
# Exports compact CSV summaries (details + raw) and keeps at most KEEP .ncu-rep
# files, so gpurun_out/ stays under the 64 MiB merge limit.
# Usage: tools/ncu_full.sh <tag> [workload] [keep-regex]
set -u
TAG=${1:-r01}
WL=${2:-cfg2}
KEEP=${3:-^$}
OUT=gpurun_out
cap() {  # name regex skip count
  local rep="$OUT/${TAG}_$1"
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
    --kernel-name-base demangled -k "regex:$2" -s "$3" -c "$4" -o "$rep" -f \
    python tools/profile_step.py --workload "$WL" > "$rep.log" 2>&1
  echo "ncu $1 rc=$?"
  if [ -f "$rep.ncu-rep" ]; then
    ncu -i "$rep.ncu-rep" --page details --csv > "$rep.details.csv" 2>/dev/null
    ncu -i "$rep.ncu-rep" --page raw --csv > "$rep.raw.csv" 2>/dev/null
    gzip -f "$rep.raw.csv"
    if ! echo "$1" | grep -Eq "$KEEP"; then rm -f "$rep.ncu-rep"; fi
  fi
}
cap ks_inner 'ks_inner' 2 1
cap moddown_rescale 'JobModDownRescale' 0 2
cap modup 'JobModUp' 2 2
cap topu 'JobTopU' 0 2
cap invgather 'JobInvGather' 0 2
cap rot_partial 'rot_partial' 0 1
