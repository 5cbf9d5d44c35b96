#!/bin/bash
# ncu --set full captures of the key-switch kernels of a cfg3 pair batch
# (N=2^16, L=24) and of device key generation; run under gpurun (1 GPU).
# profile_step --no-align 48: only pairs without alignment rotations, so the
# first ModUp / inner-product launches are a relinearisation pair batch.
# Usage: tools/ncu_cfg3.sh <tag> [modup,ks_inner,keyfused,uni_emit]
set -u
TAG=${1:-r02}
OUT=gpurun_out
cap() {  # name regex skip count
  local rep="$OUT/${TAG}_$1"
  timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none \
    --kernel-name-base demangled -k "regex:$2" -s "$3" -c "$4" -o "$rep" -f \
    python tools/profile_step.py --workload cfg3 --no-align 48 --warmup 0 > "$rep.log" 2>&1
  echo "ncu $1 rc=$?"
  if [ -f "$rep.ncu-rep" ]; then
    ncu -i "$rep.ncu-rep" --page details --csv > "$rep.details.csv" 2>/dev/null
    ncu -i "$rep.ncu-rep" --page raw --csv > "$rep.raw.csv" 2>/dev/null
    gzip -f "$rep.raw.csv"
    rm -f "$rep.ncu-rep"
  fi
}
WHICH=${2:-modup,ks_inner,keyfused,uni_emit}
[[ $WHICH == *modup* ]] && cap modup 'JobModUp>' 0 2
[[ $WHICH == *ks_inner* ]] && cap ks_inner 'ks_inner_tma' 0 1
[[ $WHICH == *keyfused* ]] && cap keyfused 'JobKeyFused' 0 2
[[ $WHICH == *uni_emit* ]] && cap uni_emit 'pk_uni_emit' 0 1
true
