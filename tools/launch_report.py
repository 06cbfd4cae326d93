"""Launch-list report for profiles/: per-kernel launches, time, share and DRAM
bytes from an ncu CSV (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv), plus the per-class DRAM traffic JSON bench.py
reads for roofline.traffic (NTT classes = one column + one chunk kernel).
usage: python tools/launch_report.py launches.csv workload out.md out.json"""
import csv
import json
import re
import sys
from collections import defaultdict

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name)
    return re.sub(r"tg::\(anonymous namespace\)::|tg::|<unnamed>::", "", name).strip()


def main():
    path, workload, out_md, out_json = sys.argv[1:5]
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    per = defaultdict(dict)
    names = {}
    for r in csv.DictReader(lines[start:]):
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r.get("Metric Unit", ""), 1.0)
        per[r["ID"]][r["Metric Name"]] = v
        names[r["ID"]] = short(r["Kernel Name"])
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    total = sum(a[1] for a in agg.values())
    rows = sorted(agg.items(), key=lambda kv: -kv[1][1])
    md = ["| kernel | launches | ms | share | DRAM MB / launch |", "|---|---|---|---|---|"]
    for k, (n, t, b) in rows:
        md.append(f"| {k} | {n} | {t:.2f} | {t / total:.1%} | {b / n / 1e6:.1f} |")
    ntt = sum(a[1] for k, a in agg.items() if k.startswith("kw_"))
    classes = {}
    for cls, pat in (("ntt_fwd", "kw_fwd_"), ("ntt_inv", "kw_inv_")):
        ks = [a for k, a in agg.items() if k.startswith(pat)]
        if ks:
            n = sum(a[0] for a in ks)  # per kernel launch (column and chunk phases), as tg_profile_read counts
            classes[cls] = {"dram_bytes_per_launch": sum(a[2] for a in ks) / n, "launches": n}
    for cls, pat in (("mod_down", "k_mod_down"), ("key_inner", "k_key_inner_b"), ("modup_baseconv", "k_modup"),
                     ("ks_fused", "kw_ks_chunks"),
                     ("lincomb", "k_lincomb"), ("tensor", "k_tensor")):
        ks = [a for k, a in agg.items() if k.startswith(pat)]
        if ks:
            n = sum(a[0] for a in ks)
            classes[cls] = {"dram_bytes_per_launch": sum(a[2] for a in ks) / n, "launches": n}
    with open(out_md, "w") as f:
        f.write(f"# {workload}: ncu launch list of one timed step\n\n")
        f.write("Command (GPU box, after the same command exited 0 without ncu):\n"
                "`TG_PROFILE_REGION=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,"
                "dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv "
                "python bench.py --steps 1 --warmup 3 --no-cpu-baseline`\n"
                "(cold cache, kernels serialised by ncu: shares are meaningful, absolute times are not).\n\n")
        f.write("\n".join(md) + "\n\n")
        f.write(f"* NTT (kw_*): {ntt / total:.0%} of kernel time; total {total:.1f} ms serialised, "
                f"{sum(a[0] for a in agg.values())} launches.\n")
        for cls, c in classes.items():
            f.write(f"* {cls}: {c['dram_bytes_per_launch'] / 1e6:.1f} MB DRAM per launch ({c['launches']} launches)\n")
    with open(out_json, "w") as f:
        json.dump({"source": f"{path} (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                             "dram__bytes_write.sum --clock-control none, TG_PROFILE_REGION=1, bench.py --steps 1 "
                             "--warmup 3; cold-cache, serialised)", "classes": classes}, f, indent=1)
    print("\n".join(md[:14]))


if __name__ == "__main__":
    main()
