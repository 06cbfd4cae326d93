#!/usr/bin/env python3
"""Kernel microbenchmarks through the C-ABI-backed module (device time via
CUDA events on the ring's stream). Used for ncu captures and roofline
iteration on single ops: NTT fwd/inv, tensor, ModUp, key inner product,
ModDown, rescale at config-3 shapes.

  python tools/kbench.py [--rows 21] [--reps 50] [--ops ntt,modup,...]
"""
from __future__ import annotations

import argparse
import os
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
# TG_ROOT: load the package from a variant build (tools/build_variant.sh)
sys.path.insert(0, os.environ.get("TG_ROOT", str(ROOT)))


def main():
    import torch

    from paper_2412_13269_b200 import tetris as G
    from paper_2412_13269_b200 import workloads as W

    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--levels", default="20,10")
    ap.add_argument("--batch", type=int, default=1, help="polys per NTT launch")
    ap.add_argument("--ops", default="ntt,intt,relin,rescale")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--bsizes", default="1,2,4,8,16,32", help="poly counts of the batch op")
    a = ap.parse_args()
    spec = W.CONFIGS[a.config]
    S = W.make_context(G, spec)
    ring = S.ring
    ext = torch.cuda.ExternalStream(ring.stream_handle())
    res = {}

    def timeit(name, fn, nbytes=None):
        for _ in range(3):
            fn()
        ring.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        prof = os.environ.get("TG_PROFILE_REGION") == "1"  # ncu --profile-from-start off
        if prof:
            torch.cuda.cudart().cudaProfilerStart()
        e0.record(ext)
        for _ in range(a.reps):
            fn()
        e1.record(ext)
        ring.synchronize()
        if prof:
            torch.cuda.cudart().cudaProfilerStop()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        res[name] = {"us": round(ms * 1e3, 2)}
        if nbytes:
            res[name]["GBps"] = round(nbytes / (ms / 1e3) / 1e9, 1)
        print(name, res[name], flush=True)

    G.profile_enable(ring, False)
    if "batch" in a.ops:  # NTT launch cost vs rows: P polys x 21 rows in one launch
        import numpy as np
        lvl = ring.max_level()
        for P in (int(x) for x in a.bsizes.split(",")):
            arr = np.random.default_rng(P).integers(0, 1 << 40, size=(P, lvl + 1, spec.N), dtype=np.uint64)
            ct = G.ciphertext_from_numpy(ring, arr, lvl, G.Form.coeff, 1.0, G.Domain.slots, 0)

            def f():  # fresh exclusively-owned block (no memoised transform), then in-place NTT
                c = S.ev.mul_scalar(ct, 1.0, 1.0)
                c.to_eval()
            timeit(f"scalar+ntt_fwd_batch{P}_rows{P * (lvl + 1)}", f, 16 * P * (lvl + 1) * spec.N)
            timeit(f"scalar_only_batch{P}", lambda: S.ev.mul_scalar(ct, 1.0, 1.0), 16 * P * (lvl + 1) * spec.N)
    for lvl in (int(x) for x in a.levels.split(",") if x):
        K = spec.K
        rows = lvl + 1 + K
        p = G.sample_uniform(ring, lvl, K, G.Rng(1))
        pe = G.ntt_transform(p, G.Form.eval)
        if "ntt" in a.ops:
            timeit(f"ntt_fwd_l{lvl}_rows{rows}", lambda: G.ntt_transform(p, G.Form.eval), 16 * rows * spec.N)
        if "intt" in a.ops:
            timeit(f"ntt_inv_l{lvl}_rows{rows}", lambda: G.ntt_transform(pe, G.Form.coeff), 16 * rows * spec.N)
        rng = G.Rng(2)
        x = G.Ciphertext()
        x.parts = [G.sample_uniform(ring, lvl, 0, rng.split(i)) for i in range(2)]
        x.scale, x.domain, x.sk_id = spec.delta, G.Domain.slots, S.sk.id()
        if "relin" in a.ops:
            timeit(f"mul_relin_l{lvl}", lambda: S.ev.mul_relin(x, x, S.keys))
        if "rescale" in a.ops:
            timeit(f"rescale_l{lvl}", lambda: S.ev.rescale(x), 8 * spec.N * 2 * (2 * lvl + 1))
        if "relinb" in a.ops:  # batched (8 record blocks, part-major stack) mul_relin + rescale, per class
            xs = []
            for b in range(8):
                c = G.Ciphertext()
                c.parts = [G.sample_uniform(ring, lvl, 0, rng.split(100 + 2 * b + i)) for i in range(2)]
                c.scale, c.domain, c.sk_id = spec.delta, G.Domain.slots, S.sk.id()
                xs.append(c)
            xb = G.stack_ciphertexts(xs)
            timeit(f"mul_relin_rescale_batch8_l{lvl}", lambda: S.ev.rescale(S.ev.mul_relin(xb, xb, S.keys)))
            G.profile_enable(ring, True)
            for _ in range(5):
                S.ev.rescale(S.ev.mul_relin(xb, xb, S.keys))
            ring.synchronize()
            pr = G.profile_read(ring)
            G.profile_enable(ring, False)
            tot = sum(v[0] for v in pr.values()) / 5
            for k, v in sorted(pr.items(), key=lambda kv: -kv[1][0]):
                if v[1]:
                    print(f"  batch8 l{lvl} {k}: {v[0] / 5 * 1e3:.1f} us ({v[0] / 5 / tot * 100:.0f}%), launches {v[1] // 5}, "
                          f"{v[2] / v[1] / (v[0] / v[1] / 1e3) / 1e9:.0f} GB/s", flush=True)
        if "prof" in a.ops:
            G.profile_enable(ring, True)
            for _ in range(5):
                S.ev.mul_relin(x, x, S.keys)
            ring.synchronize()
            pr = G.profile_read(ring)
            G.profile_enable(ring, False)
            for k, v in sorted(pr.items(), key=lambda kv: -kv[1][0]):
                print(f"  relin l{lvl} {k}: {v[0] / 5 * 1e3:.1f} us/call-set, launches {v[1] // 5}, "
                      f"{v[2] / v[1] / (v[0] / v[1] / 1e3) / 1e9:.0f} GB/s", flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
