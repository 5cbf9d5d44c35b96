"""Per-step device times of one workload (CUDA events), to see run-to-run spread."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402


def main(workload="cfg3s", steps=5):
    import paper_2604_11659_b200 as pkg
    from paper_2604_11659_b200 import engine
    from paper_2604_11659_b200._lib import lib
    wl = bench.WORKLOADS[workload]
    params, ctx, keys, a, b, ea, eb, pairs, mc = bench.make_inputs(pkg, wl)
    st = torch.cuda.current_stream()
    for i in range(int(steps)):
        g0 = lib().hs_keys_generated(ctx.handle)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(st)
        engine.spmm_csr_csc(ea, eb, ctx, keys, engine.OpCounter(), mc)
        e1.record(st)
        torch.cuda.synchronize()
        print(f"step {i}: {e0.elapsed_time(e1):.1f} ms (wall {1e3 * (time.perf_counter() - t0):.1f}), "
              f"keys generated {lib().hs_keys_generated(ctx.handle) - g0}", flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
