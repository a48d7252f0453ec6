"""Aggregate ncu SASS-page stall samples by instruction range (development aid).

    ncu -i rep.ncu-rep --page source --csv > sass.csv
    python tools/sass_regions.py sass.csv 0:600 600:7260 ...
"""
import csv
import sys


def main(path, ranges):
    rows = list(csv.reader(open(path)))
    start = 2 if rows[0][0] == "Kernel Name" else 1
    h = rows[start - 1]
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    R = rows[start:]
    tot = sum(int(r[h.index("Warp Stall Sampling (All Samples)")]) for r in R if len(r) > 3)
    for spec in ranges:
        a, b = (int(x) for x in spec.split(":"))
        agg = {c: 0 for c in cols}
        n = 0
        for r in R[a:b]:
            if len(r) < len(h):
                continue
            n += int(r[h.index("Warp Stall Sampling (All Samples)")])
            for c in cols:
                agg[c] += int(r[h.index(c)] or 0)
        top = sorted(agg.items(), key=lambda kv: -kv[1])[:7]
        print(f"[{a}:{b}] {100 * n / tot:5.1f}% of samples:",
              ", ".join(f"{k[6:]} {100 * v / max(n, 1):.0f}%" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
