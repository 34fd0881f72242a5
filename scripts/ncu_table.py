"""Per-launch table (time, DRAM bytes, SM clock, L2 hit) from an ncu --csv metrics log."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ids = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
per = collections.OrderedDict()
for r in rows[1:]:
    d = per.setdefault(r[ids], {})
    d[r[mi]] = float(r[vi].replace(",", ""))
    d["k"] = r[ki]
pat = sys.argv[2] if len(sys.argv) > 2 else ""
for i, d in per.items():
    if pat not in d["k"]:
        continue
    print(f"{i:>4} {d['k'][:48]:48s} t={d.get('gpu__time_duration.sum', 0) / 1e6:6.3f}ms "
          f"rd={d.get('dram__bytes_read.sum', 0) / 1e9:6.2f}GB wr={d.get('dram__bytes_write.sum', 0) / 1e9:5.2f}GB "
          f"clk={d.get('sm__cycles_elapsed.avg.per_second', 0) / 1e9:5.2f}GHz l2hit={d.get('lts__t_sector_hit_rate.pct', 0):5.1f}%")
