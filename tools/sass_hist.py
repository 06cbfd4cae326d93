"""Static SASS instruction histogram of selected kernels (cuobjdump -sass of
the in-tree objects): opcode counts, FP64 share, and FP64 instructions per
butterfly where the kernel is an NTT phase. Usage:
  python tools/sass_hist.py [pattern ...] > profiles/r02_sass_hist.md"""
import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OBJS = sorted((ROOT / "build" / "tetris_b200").glob("*.cu.o"))
FP64 = {"DADD", "DMUL", "DFMA", "DSETP", "DMNMX", "DADD.RZ"}


def kernels(obj):
    out = subprocess.run(["cuobjdump", "-sass", str(obj)], capture_output=True, text=True).stdout
    cur, body = None, []
    for ln in out.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
        elif cur and re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
            body.append(ln)
    if cur:
        yield cur, body


def hist(body):
    c = collections.Counter()
    for ln in body:
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)((?:\.[A-Z0-9_]+)*)", ln)
        if m:
            c[m.group(1)] += 1
    return c


def main():
    pats = sys.argv[1:] or ["kw_fwd_cols2ILi8ELi8", "kw_inv_cols2ILi8ELi8", "kw_ks_chunksILi8", "kw_inv_chunksILi8",
                            "kw_fwd_chunksILi8", "k_modup", "k_mod_down_fp"]
    print("| kernel | total | FP64 (DADD/DMUL/DFMA/DSETP) | FP64 % | LDS | STS | LDG | STG | LDGSTS | UTMALDG | IMAD | top opcodes |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for obj in OBJS:
        for name, body in kernels(obj):
            if not any(p in name for p in pats):
                continue
            c = hist(body)
            tot = sum(c.values())
            fp = sum(v for k, v in c.items() if k in FP64)
            top = ", ".join(f"{k} {v}" for k, v in c.most_common(8))
            short = re.sub(r"_ZN2tg\w*?_GLOBAL__N__\w+?_\d+", "", name)[:60]
            print(f"| {short} | {tot} | {fp} | {100 * fp / max(tot, 1):.1f} | {c['LDS']} | {c['STS']} | {c['LDG']} | "
                  f"{c['STG']} | {c['LDGSTS']} | {c['UTMALDG']} | {c['IMAD']} | {top} |")


if __name__ == "__main__":
    main()
