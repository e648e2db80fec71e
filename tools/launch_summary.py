"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel
name, launches, total and mean duration (us)."""
import collections
import csv
import sys


def summarise(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        v = v / 1000 if unit in ("ns", "nsecond") else v * 1000 if unit in ("ms", "msecond") else v
        agg[d["Kernel Name"][:70]][0] += 1
        agg[d["Kernel Name"][:70]][1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"total {tot:.1f} us over {sum(a[0] for a in agg.values())} launches")
    print(f"{'us total':>10} {'n':>4} {'us mean':>9}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{t:10.1f} {n:4d} {t / n:9.1f}  {k}")


if __name__ == "__main__":
    summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
