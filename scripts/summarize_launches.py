"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: share of
device time per kernel (cold-cache, serialised launches: compare SHARES)."""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        agg[r[ki].split("(")[0][:80]].append(float(r[vi].replace(",", "")) * scale[r[ui]])
    tot = sum(sum(v) for v in agg.values())
    print(f"# {path}: {sum(len(v) for v in agg.values())} launches, {tot / 1e3:.2f} ms total device time")
    print(f"{'share':>7} {'launches':>8} {'avg_us':>10}  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{sum(v) / tot * 100:6.2f}% {len(v):8d} {sum(v) / len(v):10.1f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
