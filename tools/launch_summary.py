"""Summarise an ncu launch list (gpu__time_duration per launch) by kernel name.

    python tools/launch_summary.py gpurun_out/launches.csv [--iters N]
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 1
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        name = r[4].split("(")[0][:70]
        tot[name] += float(r[-1].replace(",", ""))
        cnt[name] += 1
    T = sum(tot.values())
    print(f"{path}: {len(rows)} launches, {T / 1e3 / iters:.1f} us per iteration ({iters} iterations)")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:20]:
        print(f"  {v / T * 100:5.1f}%  {v / 1e3 / iters:9.1f} us/iter  x{cnt[k] / iters:.0f}  {k}")


if __name__ == "__main__":
    main()
