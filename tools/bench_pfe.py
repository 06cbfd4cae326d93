"""PFE scoring + ring repacking timing on the reference
profile's small ring (profile.hpp:112-119: chain {q0 55-bit, p 54-bit special},
base-2^30 gadget, h = 2n/3): one full repack batch of N records x 8 scoring
functions. Device (eval_scores: one launch; repack: one batched key switch
per round) vs the compiled reference on one host thread; residues compared.
Prints one JSON line per N."""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from common import load_ref  # noqa: E402


def setup(T, N, m, seed=7):
    q0 = list(T.find_ntt_primes(55, 1, 2 * N))
    p = list(T.find_ntt_primes(54, 1, 2 * N, q0))
    ring = T.RingParams(N, q0 + p, 1)
    ctx = T.KeyContext(ring, T.NoiseParams(3.2, 2 * N // 3), T.GadgetVector(1, 30))
    rng = T.Rng(seed)
    sk, _ = ctx.keygen(rng)
    keys = T.gen_repack_keys(ctx, sk, rng.split(1))
    g = np.random.Generator(np.random.PCG64(seed))
    tvs = []
    for c in range(m):
        s = T.FunctionSpec()
        s.lo, s.hi = 0.0, 256.0
        s.table = list(np.round(g.uniform(0, 4, N)))
        tvs.append(T.build_test_vector(ctx, s, sk, 2.0 ** 43, rng.split(10 + c)))
    rows = g.integers(0, 256, size=(N, m)).astype(float).tolist()
    return dict(ring=ring, ctx=ctx, sk=sk, keys=keys, tvs=tvs, rows=rows)


def main():
    from paper_2412_13269_b200 import tetris as G
    R = load_ref()
    for N in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1024,4096").split(",")]:
        m = 8
        S = setup(G, N, m)
        line = {"N": N, "records": N, "functions": m}
        for rep in range(2):  # warm + timed
            S["ring"].synchronize()
            t0 = time.perf_counter()
            scores, _ = G.eval_scores(S["rows"], S["tvs"])
            S["ring"].synchronize()
            t1 = time.perf_counter()
            packed, nauto = G.repack(S["ctx"], scores, S["keys"])
            S["ring"].synchronize()
            t2 = time.perf_counter()
        line.update(gpu_eval_scores_ms=round((t1 - t0) * 1e3, 2), gpu_repack_ms=round((t2 - t1) * 1e3, 2),
                    automorphisms=nauto)
        if R is not None:
            SR = setup(R, N, m)
            t0 = time.perf_counter()
            rs, _ = R.eval_scores(SR["rows"], SR["tvs"])
            t1 = time.perf_counter()
            rp, rn = R.repack(SR["ctx"], rs, SR["keys"])
            t2 = time.perf_counter()
            line.update(ref_eval_scores_ms=round((t1 - t0) * 1e3, 1), ref_repack_ms=round((t2 - t1) * 1e3, 1),
                        bit_exact=bool(rn == nauto and all(np.array_equal(a.to_numpy(), b.to_numpy())
                                                           for a, b in zip(packed.parts, rp.parts))))
            line["speedup_total"] = round((line["ref_eval_scores_ms"] + line["ref_repack_ms"]) /
                                          (line["gpu_eval_scores_ms"] + line["gpu_repack_ms"]), 1)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
