"""Run bench.py's roofline probe once (cfg2 context), for an ncu capture of
the same NTT pass launches:  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum --csv --log-file gpurun_out/roofline_ncu.csv python tools/roofline_probe.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    import paper_2604_11659_b200 as pkg
    wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
    params = pkg.build_params(wl["ring_degree"], wl["scale_bits"], wl["levels"], wl["seed"])
    ctx = pkg.CkksContext(params)
    print(json.dumps(bench.roofline_probe(pkg, ctx, params, bench.load_peaks(), reps=1)))


if __name__ == "__main__":
    main()
