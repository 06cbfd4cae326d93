#!/usr/bin/env python3
"""Generates the golden fixtures under tests/golden/ by running the COMPILED,
UNMODIFIED reference (oracle/_ref/tetris_ref, built from
/root/reference/proj/include by oracle/Makefile). The reference ships no known-
answer vectors, so these are the pin for the CPU restatement
(tests/test_oracle_golden.py) and for the GPU path (tests/test_gpu_golden.py).

Run here (needs /root/reference at build time): python tests/golden/gen_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from common import load_ref, make_setup  # noqa: E402

R = load_ref()
assert R is not None, "build oracle/_ref first (make -C oracle reference)"


def ct_dict(prefix, ct, out):
    for i, p in enumerate(ct.parts):
        out[f"{prefix}_p{i}"] = p.to_numpy()
    out[f"{prefix}_meta"] = np.array([ct.level(), int(ct.form()), int(ct.domain), len(ct.parts)], np.int64)
    out[f"{prefix}_scale"] = np.array([ct.scale, ct.noise_bound], np.float64)
    out[f"{prefix}_skid"] = np.array([ct.sk_id], np.uint64)


def key_dict(prefix, key, out):
    out[f"{prefix}_b"] = np.stack([p.to_numpy() for p in key.b])
    out[f"{prefix}_a"] = np.stack([p.to_numpy() for p in key.a])
    out[f"{prefix}_ids"] = np.array([key.from_id, key.to_id, key.a_seed], np.uint64)


def gen_ring():
    for N in (64, 1024):
        primes = list(R.find_ntt_primes(50, 4, 2 * N))
        sp = list(R.find_ntt_primes(60, 2, 2 * N, primes))
        ring = R.RingParams(N, primes + sp, 2)
        out = {"N": np.array([N]), "moduli": np.array(primes + sp, np.uint64), "K": np.array([2])}
        for i in range(6):
            t = ring.tables(i)
            for k in ("w", "w_shoup", "winv", "winv_shoup"):
                out[f"t{i}_{k}"] = np.asarray(t[k])
            out[f"t{i}_scalars"] = np.array([t["psi"], t["n_inv"], t["n_inv_shoup"]], np.uint64)
        out["eval_exp"] = ring.eval_exp_table()
        out["slot_of_exp"] = ring.slot_of_exp_table()
        p = R.sample_uniform(ring, 3, 2, R.Rng(11))
        out["x"] = p.to_numpy()
        e = R.ntt_transform(p, R.Form.eval)
        out["x_ntt"] = e.to_numpy()
        out["x_auto5"] = R.automorphism_apply(p, 5).to_numpy()
        out["x_auto_conj"] = R.automorphism_apply(p, 2 * N - 1).to_numpy()
        out["x_ntt_auto25"] = R.automorphism_apply(e, 25).to_numpy()
        y = R.sample_uniform(ring, 3, 0, R.Rng(12))
        out["y"] = y.to_numpy()
        out["y_rescale"] = R.rescale_round(y).to_numpy()
        # sampler streams (host producers, ring.hpp:442-487)
        g = R.sample_gaussian(ring, 3.2, 1, 0, R.Rng(13))
        out["gauss"] = g.to_numpy()
        tern = R.sample_ternary_hw(ring, N // 4, 1, 0, R.Rng(14))
        out["ternary"] = tern.to_numpy()
        np.savez_compressed(HERE / f"ring_N{N}.npz", **out)


def gen_eval():
    S = make_setup(R, N=64, nq=8, K=2, group_size=2, seed=47, rotations=(1, 2, 3, 4, 8, 16), conj=True)
    out = {"N": np.array([64]), "moduli": np.array(S.primes + S.sp, np.uint64), "K": np.array([2]),
           "group": np.array([2]), "seed": np.array([47]), "h": np.array([32])}
    out["sk_coeffs"] = np.array(S.sk.coeffs(), np.int64)
    out["sk_id"] = np.array([S.sk.id()], np.uint64)
    key_dict("rlk", S.keys.relin, out)
    gexps = list(S.keys.galois_exponents())
    out["gexps"] = np.array(gexps, np.uint64)
    for g in gexps:
        key_dict(f"gk{g}", S.keys.galois_key(g), out)
    enc = R.Encoder(S.ring, 32)
    vals = [np.sin(0.37 * i) for i in range(32)]
    x = S.ctx.encrypt(S.sk, enc.encode_slots([complex(v) for v in vals], 2.0 ** 45, 7), 2.0 ** 45, R.Rng(5),
                      R.Domain.slots)
    y = S.ctx.encrypt(S.sk, enc.encode_slots([complex(0.5 - v) for v in vals], 2.0 ** 45, 5), 2.0 ** 45, R.Rng(6),
                      R.Domain.slots)
    ct_dict("x", x, out)
    ct_dict("y", y, out)
    # keyswitch pieces at levels 7 / 4 / 0
    for lvl in (7, 4, 0):
        d = R.sample_uniform(S.ring, lvl, 0, R.Rng(200 + lvl))
        out[f"d{lvl}"] = d.to_numpy()
        digs = S.ctx.decompose(d)
        out[f"d{lvl}_digits"] = np.stack([g.to_numpy() for g in digs])
        k0, k1 = S.ctx.ks_inner(digs, S.keys.relin)
        out[f"d{lvl}_ks0"], out[f"d{lvl}_ks1"] = k0.to_numpy(), k1.to_numpy()
        xs = R.sample_uniform(S.ring, lvl, 2, R.Rng(300 + lvl))
        out[f"md{lvl}_in"] = xs.to_numpy()
        out[f"md{lvl}_out"] = S.ctx.mod_down_p(xs).to_numpy()
    ev = S.ev
    ct_dict("mul", ev.mul(x, y), out)
    ct_dict("mul_relin", ev.mul_relin(x, y, S.keys), out)
    ct_dict("rescale", ev.rescale(x), out)
    ct_dict("add", ev.add(x, y), out)
    ct_dict("sub", ev.sub(x, y), out)
    ct_dict("mul_scalar", ev.mul_scalar(x, -0.318, 2.0 ** 45), out)
    ct_dict("add_scalar", ev.add_scalar(x, 0.75), out)
    ct_dict("add_scalar_eval", ev.add_scalar(ev.mul(x, y), -1.0), out)
    ct_dict("rotate1", ev.rotate(x, 1, S.keys), out)
    ct_dict("rotate3", ev.rotate(y, 3, S.keys), out)
    ct_dict("conjugate", ev.conjugate(x, S.keys), out)
    rng = R.Rng(59)
    coeffs = [float(int(rng.uniform(2001)) - 1000) / 4000.0 for _ in range(16)]
    out["cheb_coeffs"] = np.array(coeffs)
    ct_dict("cheb15", R.eval_chebyshev(ev, x, coeffs, S.keys), out)
    ct_dict("inner_sum", R.inner_sum(ev, x, 32, S.keys), out)
    np.savez_compressed(HERE / "eval_N64.npz", **out)


def gen_threshold():
    chain = R.build_chain(R.ThresholdParams(8, 12, [15, 15, 15], 1.0))
    lv = chain.levels_required()
    S = make_setup(R, N=64, nq=lv + 2, K=2, group_size=2, seed=303)
    enc = R.Encoder(S.ring, 16)
    d = 2.0 ** 45

    def e(vals, seed):
        return S.ctx.encrypt(S.sk, enc.encode_slots([complex(v) for v in vals], d, S.ring.max_level()), d, R.Rng(seed),
                             R.Domain.slots)

    scores = [float(min(64 + i, 144)) for i in range(16)]
    ct_s, ct_t, ct_n = e(scores, 33), e([80.0] * 16, 31), e([1.0 / 144.0] * 16, 32)
    out = {"N": np.array([64]), "moduli": np.array(S.primes + S.sp, np.uint64), "K": np.array([2]),
           "group": np.array([2]), "seed": np.array([303]), "levels_required": np.array([lv]),
           "scores": np.array(scores)}
    for i, st in enumerate(chain.stages):
        out[f"stage{i}_cheb"] = np.array(st.cheb)
        out[f"stage{i}_eval_coeffs"] = np.array(chain.eval_coeffs(i))
        out[f"stage{i}_meta"] = np.array([st.degree, st.gamma, st.upper, st.error])
    out["chain_meta"] = np.array([chain.sign_error, chain.achieved_beta])
    key_dict("rlk", S.keys.relin, out)
    ct_dict("s", ct_s, out)
    ct_dict("t", ct_t, out)
    ct_dict("norm", ct_n, out)
    o1 = R.eval_private_threshold(S.ev, ct_s, ct_t, ct_n, chain, S.keys)
    o2 = R.eval_private_threshold_plain_norm(S.ev, ct_s, ct_t, 1.0 / 144.0, chain, S.keys)
    ct_dict("out_enc_norm", o1, out)
    ct_dict("out_plain_norm", o2, out)
    out["decoded_plain_norm"] = np.array(enc.decode_slots(S.ctx.decrypt(S.sk, o2), o2.scale))
    np.savez_compressed(HERE / "threshold_N64.npz", **out)


if __name__ == "__main__":
    gen_ring()
    gen_eval()
    gen_threshold()
    for f in sorted(HERE.glob("*.npz")):
        print(f.name, f.stat().st_size)
