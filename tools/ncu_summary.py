"""Compact summary of an `ncu --page raw --csv` export (one row per kernel):
duration, issue/occupancy, pipe utilisation, DRAM traffic and top stalls."""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "dur"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "fmaheavy%"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("smsp__inst_executed.sum", "warp_instr"),
]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    u = dict(zip(hdr, units))
    print("| kernel | " + " | ".join(f"{s} ({u.get(k, '')})" for k, s in KEYS) + " | top stalls (per issue) |")
    print("|---" * (len(KEYS) + 2) + "|")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        st = [k for k in hdr if k.startswith("smsp__average_warps_issue_stalled_") and
              k.endswith("_per_issue_active.ratio")]
        top = sorted(((float(d[k].replace(",", "") or 0), k) for k in st), reverse=True)[:3]
        stalls = ", ".join(f"{k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]} {v:.2f}"
                           for v, k in top)
        name = d.get("Kernel Name", "")[:70].replace("|", "/")
        print(f"| {name} | " + " | ".join(d.get(k, "") for k, _ in KEYS) + f" | {stalls} |")


if __name__ == "__main__":
    main(sys.argv[1])
