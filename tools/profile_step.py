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
    ap.add_argument("--no-align", type=int, default=0,
                    help="run only the first N pairs whose operands need no alignment rotation "
                         "(pair-batch kernels only, for targeted ncu captures)")
    args = ap.parse_args()
    import paper_2604_11659_b200 as pkg
    from paper_2604_11659_b200 import engine
    wl = bench.WORKLOADS[args.workload]
    params, ctx, keys, a, b, ea, eb, pairs, mc = bench.make_inputs(pkg, wl)
    if args.no_align:
        sub = pairs[pairs[:, 2] == pairs[:, 3]][: args.no_align]

        def run():
            engine.run_pairs(ea, eb, ctx, keys, engine.OpCounter(), mc, sub)
    else:
        def run():
            engine.spmm_csr_csc(ea, eb, ctx, keys, engine.OpCounter(), mc)
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    run()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
