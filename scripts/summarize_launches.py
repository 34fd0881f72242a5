"""Summarise an `ncu --metrics gpu__time_duration.sum[,...] --csv` launch list: share of
device time per kernel (cold-cache, serialised launches: compare SHARES), plus the
per-launch averages of any other metrics collected (DRAM bytes, SM clock, tensor-pipe
activity)."""
import collections
import csv
import re
import sys

TIME = "gpu__time_duration.sum"
SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def kernel_key(name):
    # keep template arguments (they name the GEMM variant), drop the parameter list
    name = re.sub(r"\(CUtensorMap.*$", "", name)
    name = re.sub(r"\((?!int\)|bool\)).*$", "", name) if "<" not in name else name
    return name.replace("(int)", "").replace("(bool)", "")[:90]


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ii, ki = hdr.index("ID"), hdr.index("Kernel Name")
    mi, vi, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    launches = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        if r[mi] == TIME:
            v *= SCALE[r[ui]]
        launches[r[ii]][r[mi]] = v
        names[r[ii]] = kernel_key(r[ki])
    agg = collections.defaultdict(list)
    for i, m in launches.items():
        agg[names[i]].append(m)
    extra = sorted({k for m in launches.values() for k in m} - {TIME})
    tot = sum(m[TIME] for m in launches.values())
    print(f"# {path}: {len(launches)} launches, {tot / 1e3:.2f} ms total device time")
    print(f"{'share':>7} {'launches':>8} {'avg_us':>10}  " + "".join(f"{e.split('.')[0][-24:]:>26}" for e in extra)
          + "  kernel")
    for k, ms in sorted(agg.items(), key=lambda kv: -sum(m[TIME] for m in kv[1])):
        t = sum(m[TIME] for m in ms)
        cols = "".join(f"{sum(m.get(e, 0.0) for m in ms) / len(ms):26.4g}" for e in extra)
        print(f"{t / tot * 100:6.2f}% {len(ms):8d} {t / len(ms):10.1f}  {cols}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
