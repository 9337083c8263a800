"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel.

usage: python scripts/launch_summary.py gpurun_out/launches.csv [first_id last_id]
"""
import collections
import csv
import sys

UNIT = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}


def load(path, lo=0, hi=10**9):
    rows = list(csv.reader(open(path)))
    hi_row = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi_row]
    ki, vi, ui, ii = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
    gi, bi = h.index("Grid Size"), h.index("Block Size")
    out = []
    for r in rows[hi_row + 1:]:
        if len(r) <= vi or not r[ii].isdigit():
            continue
        i = int(r[ii])
        if not (lo <= i <= hi):
            continue
        out.append((i, r[ki], float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0), r[gi], r[bi]))
    return out


def main():
    path = sys.argv[1]
    lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, 10**9)
    launches = load(path, lo, hi)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for _, name, us, _, _ in launches:
        k = name.split("(")[0]
        agg[k][0] += 1
        agg[k][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{len(launches)} launches, {tot / 1e3:.3f} ms total (serialised, cold-cache)")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t / 1e3:9.3f} ms {100 * t / tot:5.1f}% {n:6d} x {t / n:8.2f} us  {k[:90]}")


if __name__ == "__main__":
    main()
