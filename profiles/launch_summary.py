"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel name, launches and mean/total device time (cold-cache, serialised:
compare SHARES of the step, not absolutes)."""
import collections
import csv
import sys


def main(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0][:70]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':72s} {'n':>4s} {'mean_us':>9s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:72s} {n:4d} {t / n / 1e3:9.1f} {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        main(p)
