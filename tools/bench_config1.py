"""Config 1 (BASELINE.json configs[0]): the CKKS ring-op microbench.
N = 2^14, 8 x 50-bit q, 2 x 60-bit P, group 2 (dnum 4), h = 192, 64 ciphertexts
of uniform residues from a seed. Ops: forward / inverse NTT of every part,
tensor + relinearisation of ct_i x ct_{i+1 mod 64}, rescale, rotation by 1 -
each as ONE batched device op over the 64 ciphertexts. Algorithmic bytes per
SURVEY 8(d) (config-1 totals). The reference (one host thread) runs the same
ops on a 4-ciphertext sample, compared residue for residue, and its time is
scaled to 64 ciphertexts. Prints one JSON line."""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from common import load_ref  # noqa: E402

MIB = 1 << 20


def build(T, spec, n_cts):
    from paper_2412_13269_b200 import workloads as W
    S = W.make_context(T, spec, rotations=(1,))
    rng = T.Rng(spec.seed).split(5)
    L = S.ring.max_level()
    cts = []
    for i in range(n_cts):
        c = T.Ciphertext()
        c.parts = [T.sample_uniform(S.ring, L, 0, rng.split(2 * i + j)) for j in range(2)]
        c.scale, c.domain, c.sk_id = spec.delta, T.Domain.slots, S.sk.id()
        cts.append(c)
    return S, cts


def main():
    from paper_2412_13269_b200 import tetris as G
    from paper_2412_13269_b200 import workloads as W
    spec = W.CONFIGS[1]
    n = spec.n_cts
    S, cts = build(G, spec, n)
    ev, keys, ring = S.ev, S.keys, S.ring
    fat = G.stack_ciphertexts(cts)
    nxt = G.stack_ciphertexts(cts[1:] + cts[:1])
    limb = spec.N * 8
    L1 = spec.nq  # limbs per part
    fat_eval = fat.copy()
    fat_eval.to_eval()

    def fresh(c):  # an exclusively owned copy (mul by 1): the transform below is real, not memoised
        return ev.mul_scalar(c, 1.0, 1.0)

    def fwd():
        c = fresh(fat)
        c.to_eval()
        return c

    def inv():
        c = fresh(fat_eval)
        c.to_coeff()
        return c

    ntt_bytes = 2 * n * L1 * limb * 2  # every part read + written once
    ops = {
        "scalar_copy": (lambda: fresh(fat), 2 * n * L1 * limb * 2),
        "ntt_fwd": (fwd, ntt_bytes),
        "ntt_inv": (inv, ntt_bytes),
        "tensor_relin": (lambda: ev.mul_relin(fat, nxt, keys), None),
        "rescale": (lambda: ev.rescale(fat), None),
        "rotate_1": (lambda: ev.rotate(fat, 1, keys), None),
    }
    res = {"config": spec.name, "ciphertexts": n, "N": spec.N, "q_limbs": L1, "special": spec.K,
           "dnum": -(-spec.nq // spec.group)}
    outs = {}
    for name, (fn, alg) in ops.items():
        for _ in range(3):
            o = fn()
        ring.synchronize()
        reps = 20
        t0 = time.perf_counter()
        for _ in range(reps):
            o = fn()
        ring.synchronize()
        us = (time.perf_counter() - t0) / reps * 1e6
        outs[name] = o
        res[name] = {"us_64cts": round(us, 1)}
        if alg:
            res[name]["GBps"] = round(alg / (us / 1e6) / 1e9, 1)
    for name in ("ntt_fwd", "ntt_inv"):  # net of the copy that makes the block exclusive
        net = res[name]["us_64cts"] - res["scalar_copy"]["us_64cts"]
        res[name]["net_us_64cts"] = round(net, 1)
        res[name]["net_GBps"] = round(ntt_bytes / (net / 1e6) / 1e9, 1)
    R = load_ref()
    if R is not None:
        k = 4
        SR, rcts = build(R, spec, k)
        ref = {}
        t0 = time.perf_counter()
        ref["tensor_relin"] = [SR.ev.mul_relin(rcts[i], rcts[(i + 1) % k], SR.keys) for i in range(k - 1)]
        ref["tensor_relin_s"] = (time.perf_counter() - t0) / (k - 1)
        t0 = time.perf_counter()
        ref["rescale"] = [SR.ev.rescale(c) for c in rcts]
        ref["rescale_s"] = (time.perf_counter() - t0) / k
        t0 = time.perf_counter()
        ref["rotate_1"] = [SR.ev.rotate(c, 1, SR.keys) for c in rcts]
        ref["rotate_1_s"] = (time.perf_counter() - t0) / k
        exact = True
        for name in ("tensor_relin", "rescale", "rotate_1"):
            got = G.unstack_ciphertext(outs[name])
            for i, rc in enumerate(ref[name]):
                exact &= all(np.array_equal(a.to_numpy(), b.to_numpy()) for a, b in zip(got[i].parts, rc.parts))
            res[name]["ref_us_64cts_1thread"] = round(ref[name + "_s"] * n * 1e6, 1)
            res[name]["speedup"] = round(res[name]["ref_us_64cts_1thread"] / res[name]["us_64cts"], 1)
        res["bit_exact_vs_reference_sample"] = bool(exact)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
