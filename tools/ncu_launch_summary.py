"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
total / count / mean microseconds per kernel name."""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def main(fn, top=25):
    hdr, agg = None, collections.defaultdict(lambda: [0.0, 0])
    for r in csv.reader(open(fn)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        us = float(d["Metric Value"].replace(",", "")) * SCALE.get(d.get("Metric Unit", "ns"), 1e-3)
        k = d["Kernel Name"][:70]
        agg[k][0] += us
        agg[k][1] += 1
    tot = sum(v[0] for v in agg.values())
    for k, (t, n) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{t:10.1f} us {100 * t / tot:5.1f}%  n={n:5d}  avg={t / n:8.2f} us  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
