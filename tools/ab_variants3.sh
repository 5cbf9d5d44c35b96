#!/bin/bash
# interleaved A/B: tools/ab_variants3.sh <tag> <workload> <rounds> <variant>...
TAG=$1; WL=$2; R=$3; shift 3
for r in $(seq $R); do for v in "$@"; do
  if [ "$v" = default ]; then unset HS_LIB_PATH; else export HS_LIB_PATH=$PWD/paper_2604_11659_b200/lib/variants/$v.so; fi
  timeout 900 python bench.py --workload $WL --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/${TAG}_${WL}_${v}_$r.json 2>/dev/null
  echo "$WL $v $r $(python -c "import json;print(json.load(open('gpurun_out/${TAG}_${WL}_${v}_$r.json'))['ms_per_step'])" 2>&1)"
done; done
unset HS_LIB_PATH
