"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_summary.py profiles/r01_launches_v5.csv
"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    head, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            head = r
            continue
        if head and len(r) == len(head):
            d = dict(zip(head, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0].replace("bx::<unnamed>::", "").replace("<unnamed>::", "")
                data.append((name, float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)))
    agg = collections.OrderedDict()
    for k, v in data:
        agg.setdefault(k, []).append(v)
    print(f"{'kernel':58s} {'launches':>8s} {'mean us':>10s} {'total us':>10s}")
    for k, v in agg.items():
        print(f"{k[:58]:58s} {len(v):8d} {sum(v) / len(v):10.1f} {sum(v):10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
