"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv
--log-file X) by kernel: launches, total and mean time, share.
usage: python tools/launch_agg.py launches.csv [steps]"""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"tg::\(anonymous namespace\)::|tg::", "", name)
    return name


def main():
    path = sys.argv[1]
    steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v *= {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
        a = agg[short(r["Kernel Name"])]
        a[0] += 1
        a[1] += v
    total = sum(a[1] for a in agg.values())
    print(f"| kernel | launches/step | ms/step | mean us | share |\n|---|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {n / steps:.0f} | {t / steps / 1e3:.2f} | {t / n:.1f} | {t / total:.1%} |")
    print(f"| total | {sum(a[0] for a in agg.values()) / steps:.0f} | {total / steps / 1e3:.2f} | | |")


if __name__ == "__main__":
    main()
