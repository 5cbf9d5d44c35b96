#!/bin/bash
# A/B of library variants (tools/build_variant.sh) on one bench workload, 3 timed steps each:
# tools/ab_variants.sh <tag> <workload> <variant>... ("default" = the in-tree build)
TAG=$1; WL=$2; shift 2
for v in "$@"; do
  if [ "$v" = default ]; then unset HS_LIB_PATH; else export HS_LIB_PATH=$PWD/paper_2604_11659_b200/lib/variants/$v.so; fi
  timeout 900 python bench.py --workload $WL --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/${TAG}_${WL}_$v.json 2> gpurun_out/${TAG}_${WL}_$v.err
  echo "$WL $v rc=$? $(python -c "import json;print(json.load(open('gpurun_out/${TAG}_${WL}_$v.json'))['ms_per_step'])" 2>&1)"
done
unset HS_LIB_PATH
