"""Per-kernel totals of an ncu launch list (`--metrics gpu__time_duration.sum --csv`).
Usage: python tools/launch_table.py launches.csv"""
import collections
import csv
import sys

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def main(path):
    h, agg = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "ID":
            h = r
            continue
        if h is None or r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        v = float(r[h.index("Metric Value")].replace(",", "")) * UNIT[r[h.index("Metric Unit")]]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {n} | {t:.2f} | {100 * t / tot:.1f}% |")
    print(f"| total | | {tot:.2f} | |")


if __name__ == "__main__":
    main(sys.argv[1])
