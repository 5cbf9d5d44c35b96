#!/bin/bash
# Round-2 final measurements: the driver's commands on the final build.
T=r02z
python -m pytest tests -m gpu -x -q > gpurun_out/${T}_gputest.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${T}_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke rc=$?
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench_cfg3_driver_cmd.json 2> gpurun_out/${T}_bench_cfg3_driver_cmd.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench_reference_driver_cmd.json 2> gpurun_out/${T}_bench_reference.err; echo ref rc=$?
python tools/ntt_micro.py > gpurun_out/${T}_ntt_micro.log 2>&1
python tools/keygen_micro.py > gpurun_out/${T}_keygen_micro.log 2>&1
cut -c1-300 gpurun_out/${T}_bench_cfg3_driver_cmd.json
