#!/bin/bash
# A/B of library variants (tools/build_variant.sh) on one bench workload:
# tools/ab_cfg3.sh <tag> <workload> <variant>... ("default" = the in-tree build)
TAG=$1; WL=$2; shift 2
for v in "$@"; do
  if [ "$v" = default ]; then unset HS_LIB_PATH; else export HS_LIB_PATH=$PWD/paper_2604_11659_b200/lib/variants/$v.so; fi
  timeout 900 python bench.py --workload $WL --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_$v.json 2> gpurun_out/${TAG}_$v.err
  echo "$v rc=$?"
done
unset HS_LIB_PATH
