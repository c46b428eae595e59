"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import re
import sys


def main(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rd = csv.DictReader(lines)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in rd:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(unsigned.*$|\(.*$", "", d["Kernel Name"]).replace("void ", "")
        name = name.replace("<unnamed>::", "")
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[d["Metric Unit"]]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':40s} {'launches':>8s} {'ms':>9s} {'share':>6s}")
    for k, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:40s} {c:8d} {us / 1e3:9.3f} {100 * us / tot:5.1f}%")
    print(f"{'total':40s} {sum(v[0] for v in agg.values()):8d} {tot / 1e3:9.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
