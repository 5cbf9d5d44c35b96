"""Micro-benchmark of the batched NTT kernel (CUDA events), for A/B tuning."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_11659_b200 as P
from paper_2604_11659_b200 import device as D
from paper_2604_11659_b200._lib import check, lib

for log_n, L, items in [(14, 2, 2048), (16, 2, 512), (16, 24, 24)]:
    n = 1 << log_n
    params = P.build_params(n, 50, L, 2024)
    ctx = P.CkksContext(params)
    limbs = items * (L + 2)
    buf = D.zeros((limbs, n))
    for inv in (0, 1):
        for _ in range(3):
            check(lib().hs_ntt(ctx.handle, D.ptr(buf), items, L + 2, 0, inv, D.stream()))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        reps = 10
        for _ in range(reps):
            check(lib().hs_ntt(ctx.handle, D.ptr(buf), items, L + 2, 0, inv, D.stream()))
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        bfly = limbs * (n // 2) * log_n
        print(f"n=2^{log_n} L={L} limbs={limbs} {'INTT' if inv else 'NTT '}: {ms:.3f} ms  "
              f"{bfly / ms / 1e6:.1f} G butterflies/s  {limbs * 32 * n / ms / 1e6:.0f} GB/s (2 passes)")
