"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list: kernel, launches, total and mean us."""
import collections
import csv
import sys


def main(path, top=15):
    hdr, agg = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(d["Metric Unit"], 1.0)
        a = agg.setdefault(d["Kernel Name"].split("(")[0][:60], [0, 0.0])
        a[0] += 1
        a[1] += v
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{k:60s} n={n:5d} total={t:12.1f} us  mean={t / n:10.2f} us")


if __name__ == "__main__":
    main(sys.argv[1])
