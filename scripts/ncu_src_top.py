"""Top stalled SASS instructions of an ncu source-page CSV (ncu -i rep --page source --csv):
address, samples, dominant stall reasons, instruction, with N lines of preceding context."""
import csv
import sys


def main(path, n=25, ctx=0):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Source" in r and "Address" in r][0]
    hdr = rows[hi]
    data, seen = [], set()
    for r in rows[hi + 1:]:
        if len(r) == len(hdr) and r[0] not in seen:
            seen.add(r[0])
            data.append(r)
    f = lambda x: float(x) if x.replace(".", "", 1).isdigit() else 0.0
    i_s, i_src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = sum(f(r[i_s]) for r in data)
    print(f"# {path}: {tot:.0f} samples")
    order = sorted(range(len(data)), key=lambda i: -f(data[i][i_s]))[:n]
    for i in order:
        r = data[i]
        rs = sorted(((f(r[hdr.index(h)]), h[6:]) for h in reasons), reverse=True)[:3]
        why = " ".join(f"{h}={v:.0f}" for v, h in rs if v > 0)
        for j in range(max(0, i - ctx), i):
            print(f"        {data[j][i_src][:80]}")
        print(f"{r[0][-6:]} {f(r[i_s]) / tot * 100:5.1f}%  {r[i_src][:60]:60s} {why}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25, int(sys.argv[3]) if len(sys.argv) > 3 else 0)
