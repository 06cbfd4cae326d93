#!/usr/bin/env python3
"""NTT microbenchmark straight through the C-ABI (include/tetris_b200.h):
tg_context_create from the config-4 ring tables, device buffers of P polys,
batched tg_ntt_forward / tg_ntt_inverse timed with CUDA events on the
launching stream. Shapes are the ones the config-4 query launches (product
inputs, ModUp digits, key-switch accumulators). Prints per case the device
time, us per row and algorithmic GB/s (16 B per coefficient), plus an output
checksum (seeded inputs) so kernel variants can be compared bit for bit, and
a forward->inverse round-trip check.

  python tools/nttbench.py [--reps 20] [--cases fwd:16:20:0,...]
"""
from __future__ import annotations

import argparse
import os
import ctypes
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
# TG_ROOT: load the package from a variant build (tools/build_variant.sh)
sys.path.insert(0, os.environ.get("TG_ROOT", str(ROOT)))

DEFAULT_CASES = "fwd:16:20:0,fwd:32:20:7,inv:16:20:7,inv:16:20:0,fwd:4:20:7,inv:2:10:7"


def main():
    import numpy as np
    import torch

    from paper_2412_13269_b200 import load_c_abi, tetris as G
    from paper_2412_13269_b200 import workloads as W

    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--cases", default=DEFAULT_CASES, help="dir:polys:level:nspecial,...")
    ap.add_argument("--config", type=int, default=4)
    a = ap.parse_args()

    spec = W.CONFIGS[a.config]
    qs, sp = W._primes(G, spec)
    ring = G.RingParams(spec.N, qs + sp, spec.K)
    N, mods = spec.N, qs + sp
    tabs = np.empty((len(mods), 4, N), dtype=np.uint64)
    ninv = np.empty((len(mods), 2), dtype=np.uint64)
    for i in range(len(mods)):
        t = ring.tables(i)
        tabs[i] = [t["w"], t["w_shoup"], t["winv"], t["winv_shoup"]]
        ninv[i] = [t["n_inv"], t["n_inv_shoup"]]
    ee = np.ascontiguousarray(ring.eval_exp_table(), dtype=np.uint32)
    se = np.ascontiguousarray(ring.slot_of_exp_table(), dtype=np.uint32)
    L = load_c_abi()
    print("library:", L._name, flush=True)
    P64, P32, VP = ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32), ctypes.c_void_p
    ctx = VP()
    moda = np.array(mods, dtype=np.uint64)
    rc = L.tg_context_create(ctypes.byref(ctx), 0, N, moda.ctypes.data_as(P64), len(mods), spec.K,
                             tabs.ctypes.data_as(P64), ninv.ctypes.data_as(P64), ee.ctypes.data_as(P32),
                             se.ctypes.data_as(P32))
    if rc:
        raise RuntimeError(L.tg_last_error())
    L.tg_last_error.restype = ctypes.c_char_p
    dev = torch.device("cuda:0")
    stream = torch.cuda.Stream(dev)
    sh = VP(stream.cuda_stream)
    out = {}
    for case in a.cases.split(","):
        d, P, lvl, ns = case.split(":")
        P, lvl, ns = int(P), int(lvl), int(ns)
        rows = lvl + 1 + ns
        rowmods = [mods[r] if r <= lvl else mods[len(qs) + r - lvl - 1] for r in range(rows)]
        g = torch.Generator(device=dev).manual_seed(1234 + P * 100 + rows)
        with torch.cuda.stream(stream):
            x = torch.randint(0, 1 << 62, (P, rows, N), dtype=torch.int64, device=dev, generator=g)
            qt = torch.tensor([int(m) for m in rowmods], dtype=torch.int64, device=dev).view(1, rows, 1)
            x = torch.remainder(x, qt)
            y = x.clone()
        fn = L.tg_ntt_forward if d == "fwd" else L.tg_ntt_inverse
        inv = L.tg_ntt_inverse if d == "fwd" else L.tg_ntt_forward

        def run(buf):
            r = fn(ctx, VP(buf.data_ptr()), lvl, ns, P, sh)
            if r:
                raise RuntimeError(L.tg_last_error())

        run(y)  # checksum of one transform
        stream.synchronize()
        ck = int(torch.sum(y.view(-1) % 1000003).item())
        inv(ctx, VP(y.data_ptr()), lvl, ns, P, sh)
        stream.synchronize()
        rt = bool(torch.equal(x, y))
        for _ in range(3):
            run(y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream.synchronize()
        e0.record(stream)
        for _ in range(a.reps):
            run(y)
        e1.record(stream)
        stream.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / a.reps
        nrows = P * rows
        res = {"us": round(us, 1), "us_per_row": round(us / nrows, 4),
               "GBps": round(16.0 * nrows * N / (us * 1e-6) / 1e9, 1), "checksum": ck, "roundtrip": rt}
        out[case] = res
        print(case, res, flush=True)
        del x, y
    L.tg_context_destroy(ctx)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
