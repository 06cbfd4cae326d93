"""Aggregate ncu's SASS source page (warp-stall samples per instruction) by
opcode: where a kernel's warps wait. Usage:
  ncu -i rep --page source --csv --kernel-name regex:K --launch-skip S --launch-count 1 --print-source sass > k.csv
  python tools/ncu_sass_stalls.py k.csv"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr, data = rows[hi], [r for r in rows[hi + 1:] if len(r) == len(rows[hi]) and r[0] != "Address"]
    i_s, i_src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]

    def num(x):
        try:
            return float(x)
        except ValueError:
            return 0.0

    tot = sum(num(r[i_s]) for r in data) or 1.0
    agg, aggst = collections.Counter(), collections.defaultdict(collections.Counter)
    for r in data:
        toks = r[i_src].strip().split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        agg[op] += num(r[i_s])
        for i in stall_cols:
            aggst[op][hdr[i][6:]] += num(r[i])
    print(f"total stall samples {tot:.0f}")
    print("| opcode | share of samples | top stall reasons (samples) |")
    print("|---|---|---|")
    for op, v in agg.most_common(14):
        top = ", ".join(f"{k} {x:.0f}" for k, x in aggst[op].most_common(4) if x > 0)
        print(f"| {op} | {100 * v / tot:.1f}% | {top} |")


if __name__ == "__main__":
    main(sys.argv[1])
