"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    out = []
    for r in data:
        if len(r) <= vi or r[vi] == "":
            continue
        out.append((r[ki], float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)))
    return out


def short(name):
    m = re.match(r"(?:void )?(?:hs::)?(\w+)(<.*>)?\(", name)
    if not m:
        return name[:90]
    base = m.group(1)
    if m.group(2):
        targs = re.sub(r"hs::|, int|\(.*", "", m.group(2))
        base += targs[:80]
    return base


def main(path):
    rows = load(path)
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for name, us in rows:
        k = short(name)
        tot[k] += us
        cnt[k] += 1
    T = sum(tot.values())
    print(f"total {T / 1e3:.2f} ms over {len(rows)} launches")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v / 1e3:9.3f} ms {100 * v / T:5.1f}%  n={cnt[k]:4d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
