"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count, mean and
total device time, and share of the total.  Usage: python profiles/summarize_launches.py launches.csv"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        agg[r[ki].split("(")[0].replace("void ", "")[:48]].append(v)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':48s} {'n':>5s} {'mean_us':>9s} {'total_us':>10s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:48s} {len(v):5d} {sum(v) / len(v):9.2f} {sum(v):10.1f} {sum(v) / tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
