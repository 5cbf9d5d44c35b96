"""Histogram of executed SASS opcodes from `ncu --page source --csv --print-source sass`."""
import collections
import csv
import re
import sys


def main(path, which=0, show=0):
    blocks, cur = [], None
    for row in csv.reader(open(path)):
        if row and row[0] == "Kernel Name":
            cur = {"name": row[1], "rows": []}
            blocks.append(cur)
            continue
        if cur is None or not row or row[0] == "Address":
            continue
        cur["rows"].append(row)
    b = blocks[which]
    hist = collections.Counter()
    stall = collections.Counter()
    tot = 0
    for r in b["rows"]:
        try:
            ex = int(float(r[5] or 0))
        except ValueError:
            continue
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]+)", r[1])
        if not m:
            continue
        op = m.group(2)
        hist[op] += ex
        tot += ex
    print(b["name"][:120], f"total warp-instr {tot:,}")
    for k, v in hist.most_common(25):
        print(f"{k:10s} {v:14,d} {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
