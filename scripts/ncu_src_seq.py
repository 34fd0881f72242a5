"""Address-ordered SASS lines of an ncu source-page CSV with at least --min % of the warp
stall samples (with their top stall reasons): where in the code the samples fall."""
import csv
import sys


def main(path, thresh=0.1):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Source" in r and "Address" in r][0]
    h = rows[hi]
    d = [r for r in rows[hi + 1:] if len(r) == len(h)]
    i_s, i_src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    f = lambda x: float(x) if x.replace(".", "", 1).isdigit() else 0.0
    tot = sum(f(r[i_s]) for r in d)
    reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
    for r in d:
        s = f(r[i_s]) / tot * 100
        if s >= thresh:
            rs = sorted(((f(r[h.index(x)]), x[6:]) for x in reasons), reverse=True)[:2]
            print(r[0][-6:], f"{s:5.2f}", r[i_src][:64], " ".join(f"{b}={a:.0f}" for a, b in rs if a > 0))


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.1)
