"""profiles/gemm_traffic.json from an ncu launch list with dram__bytes_{read,write}.sum:
DRAM bytes per GEMM launch averaged over one step's GEMM launches (the same averaging as
bench.py's roofline.achieved), plus the per-variant breakdown.

    python scripts/gemm_traffic.py <launches.csv> <workload name> [profiles/gemm_traffic.json]
"""
import collections
import csv
import json
import os
import re
import sys


def main(path, workload, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ii, ki, mi, vi = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    per = collections.defaultdict(dict)
    name = {}
    for r in rows[1:]:
        if "gemm_kernel" not in r[ki]:
            continue
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        name[r[ii]] = re.sub(r"\(CUtensorMap.*$", "", r[ki]).replace("(int)", "").replace("(bool)", "")
    tot = [m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in per.values()]
    by = collections.defaultdict(list)
    for i, m in per.items():
        by[name[i]].append(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"])
    d = json.load(open(out)) if os.path.exists(out) else {}
    d[workload] = sum(tot) / len(tot)
    d.setdefault("detail", {})[workload] = {
        "source": os.path.basename(path), "launches": len(tot),
        "by_kernel_bytes_per_launch": {k: sum(v) / len(v) for k, v in by.items()},
        "note": "dram__bytes_read.sum + dram__bytes_write.sum per GEMM launch (ncu --clock-control none, "
                "serialised cold-cache replays), averaged over the GEMM launches of the profiled steps"}
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "profiles/gemm_traffic.json")
