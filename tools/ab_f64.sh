#!/bin/bash
# A/B of the FP64 forward-butterfly path (HS_NTT_F64=0 keeps every prime on
# the integer path) in one build: NTT micro-benchmark, cfg2 and cfg3s benches.
T=${1:-r02f}
for f in 1 0; do
  HS_NTT_F64=$f python tools/ntt_micro.py > gpurun_out/${T}_ntt_micro_f64$f.log 2>&1
done
for wl in cfg2 cfg3s; do
  for f in 1 0 1 0; do
    HS_NTT_F64=$f timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu-baseline \
      > gpurun_out/${T}_${wl}_f64$f.json 2> gpurun_out/${T}_${wl}_f64$f.err
    echo "$wl f64=$f rc=$? $(python -c "import json,sys;d=json.load(open('gpurun_out/${T}_${wl}_f64$f.json'));print(d['ms_per_step'])" 2>&1)"
  done
done
