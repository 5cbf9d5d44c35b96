"""One encrypted SpMSpM step between cudaProfilerStart/Stop, for ncu.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/launches.csv python tools/profile_step.py [--workload cfg2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--warmup", type=int, default=1)
    args = ap.parse_args()
    import paper_2604_11659_b200 as pkg
    from paper_2604_11659_b200 import engine
    wl = bench.WORKLOADS[args.workload]
    params, ctx, keys, a, b, ea, eb, pairs, mc = bench.make_inputs(pkg, wl)
    for _ in range(args.warmup):
        engine.spmm_csr_csc(ea, eb, ctx, keys, engine.OpCounter(), mc)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    engine.spmm_csr_csc(ea, eb, ctx, keys, engine.OpCounter(), mc)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
