"""Device Galois-key generation throughput at cfg3 parameters (N=2^16, L=24).

Times hs_key_generate_galois for K keys (CUDA events on the launch stream and
host wall clock) -- the per-key cost the runner pays inside a cfg3 step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_11659_b200 as P  # noqa: E402


def main(K=16, reps=3, log_n=16, L=24):
    params = P.build_params(1 << log_n, 50, L, 2024)
    ctx = P.CkksContext(params)
    keys = ctx.keygen()
    st = torch.cuda.current_stream()
    base = 1
    for rep in range(reps + 1):
        steps = list(range(base, base + K))      # same steps: key buffers are reused
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(st)
        k2 = ctx.gen_galois_keys(steps, keys, device=True)
        e1.record(st)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        if rep:
            print(f"K={K}: {e0.elapsed_time(e1) / K:.3f} ms/key (events), {wall * 1e3 / K:.3f} ms/key (wall)",
                  flush=True)
        del k2


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
