"""Where the end-to-end (host buffers) time of a cfg2 step goes: device-resident
step vs host-operand step vs host-operand step + result read-back."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402


def main(workload="cfg2", reps=4):
    import paper_2604_11659_b200 as pkg
    from paper_2604_11659_b200 import encmat, engine
    from paper_2604_11659_b200.types import Ciphertext
    wl = bench.WORKLOADS[workload]
    params, ctx, keys, a, b, ea, eb, pairs, mc = bench.make_inputs(pkg, wl)
    ha_t = torch.from_numpy(ea.ctxt.host()).pin_memory()
    hb_t = torch.from_numpy(eb.ctxt.host()).pin_memory()

    def run(kind):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if kind == "device":
            r = engine.spmm_csr_csc(ea, eb, ctx, keys, engine.OpCounter(), mc)
            torch.cuda.synchronize()
        else:
            ha = encmat.EncryptedSparseMatrix(Ciphertext(ha_t, ea.ctxt.scale, ea.ctxt.level), ea.meta)
            hb = encmat.EncryptedSparseMatrix(Ciphertext(hb_t, eb.ctxt.scale, eb.ctxt.level), eb.meta)
            r = engine.spmm_csr_csc(ha, hb, ctx, keys, engine.OpCounter(), mc)
            if kind == "host+d2h":
                r.ctxt.host()
            torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3

    for kind in ["device", "host", "host+d2h", "device"]:
        ts = [run(kind) for _ in range(int(reps))]
        print(f"{kind:10s} " + " ".join(f"{t:.1f}" for t in ts), flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
