"""Half-BTS (reference bootstrap.hpp) on the device vs the
compiled reference, mirroring the reference's own fixture (test_bootstrap.cpp
BtsFixture: N = 256, 55-bit q0, 45-bit working primes, a 60-bit decode prime,
three 60-bit specials, group 3, h = 32, EvalMod (30, 3, 16, 7, 0.65),
Delta_in = 2^43, Delta_evalmod = 2^45). Every stage is compared residue for
residue; slots_to_coeffs(half_bts(x)) recovers x within the reference's
2^-12 bound."""
import math

import numpy as np
import pytest

from common import assert_ct_equal

pytestmark = pytest.mark.gpu


def _fixture(T, seed, n=256, spare=2, gap=0):
    ev_cfg = T.EvalModConfig(30, 3, 16, 7, 0.65)
    tmp = T.BootstrapParams()
    tmp.evalmod, tmp.slots, tmp.sparse_log_gap, tmp.delta_input, tmp.delta_evalmod = ev_cfg, n // 2, gap, 1.0, 1.0
    depth = tmp.depth()
    q0 = list(T.find_ntt_primes(55, 1, 2 * n))
    mid = list(T.find_ntt_primes(45, depth - 1 + spare, 2 * n, q0))
    top = list(T.find_ntt_primes(60, 4, 2 * n, q0))
    chain = q0 + mid + [top[3]] + top[:3]
    ring = T.RingParams(n, chain, 3)
    ctx = T.KeyContext(ring, T.NoiseParams(3.2, 32), T.GadgetVector(3, 0))
    ev = T.Evaluator(ctx)
    p = T.BootstrapParams()
    p.slots, p.sparse_log_gap, p.secret_hw, p.evalmod = n // 2, gap, 32, ev_cfg
    p.delta_input, p.delta_evalmod = 2.0 ** 43, 2.0 ** 45
    bts = T.BootstrapEvaluator(ctx, p)
    rng = T.Rng(seed)
    sk, _ = ctx.keygen(rng)
    krng = rng.split(9)
    keys = T.EvalKeys()
    keys.relin = ctx.relin_key_gen(sk, krng)
    for g in bts.required_galois_exponents():
        if not keys.has(g):
            keys.add_galois(g, ctx.galois_key_gen(sk, g, krng))
    return dict(T=T, ring=ring, ctx=ctx, ev=ev, p=p, bts=bts, sk=sk, keys=keys)


def _encrypt_coeffs(F, v, seed):
    T = F["T"]
    enc = T.Encoder(F["ring"], F["ring"].degree() // 2)
    m = enc.encode_coeffs(list(v), F["p"].delta_input, 0)
    return F["ctx"].encrypt(F["sk"], m, F["p"].delta_input, T.Rng(seed), T.Domain.coeffs)


@pytest.fixture(scope="module")
def bts_pair(G, R, gpu_available):
    return _fixture(G, 419), _fixture(R, 419)


def _message(seed, n=256):
    g = np.random.Generator(np.random.PCG64(seed))
    return [float(x) for x in g.integers(-15, 16, n)]


def test_plans_and_exponents_match(bts_pair):
    g, r = bts_pair
    assert list(g["bts"].required_galois_exponents()) == list(r["bts"].required_galois_exponents())
    assert g["bts"].output_level() == r["bts"].output_level()


def test_half_bts_stages_bit_exact(G, bts_pair):
    g, r = bts_pair
    v = _message(5)
    cg, cr = _encrypt_coeffs(g, v, 21), _encrypt_coeffs(r, v, 21)
    rg, rr = g["bts"].mod_raise(cg), r["bts"].mod_raise(cr)
    assert_ct_equal(rg, rr, "mod_raise")
    (reg, img), (rer, imr) = g["bts"].coeffs_to_slots(g["ev"], rg, g["keys"]), r["bts"].coeffs_to_slots(r["ev"], rr, r["keys"])
    assert_ct_equal(reg, rer, "coeffs_to_slots re")
    assert_ct_equal(img, imr, "coeffs_to_slots im")
    mg, mr = g["bts"].eval_mod(g["ev"], reg, g["keys"]), r["bts"].eval_mod(r["ev"], rer, r["keys"])
    assert_ct_equal(mg, mr, "eval_mod")


def test_half_bts_round_trip(G, bts_pair):
    g, r = bts_pair
    v = _message(13)
    cg, cr = _encrypt_coeffs(g, v, 31), _encrypt_coeffs(r, v, 31)
    lg, rg_ = g["bts"].half_bts(g["ev"], cg, g["keys"])
    lr, rr_ = r["bts"].half_bts(r["ev"], cr, r["keys"])
    assert_ct_equal(lg, lr, "half_bts left")
    assert_ct_equal(rg_, rr_, "half_bts right")
    back = g["bts"].slots_to_coeffs(g["ev"], lg, rg_, g["keys"])
    back_r = r["bts"].slots_to_coeffs(r["ev"], lr, rr_, r["keys"])
    assert_ct_equal(back, back_r, "slots_to_coeffs")
    dec = g["ctx"].decrypt(g["sk"], back)
    if dec.level() > 1:
        dec.drop_to_level(1)
    got = G.Encoder(g["ring"], 128).decode_coeffs(dec, back.scale, 256)
    assert max(abs(a - b) for a, b in zip(got, v)) < 15.0 * 2.0 ** -12


def test_trace_map_bit_exact(G, R, gpu_available):
    g, r = _fixture(G, 407, gap=1), _fixture(R, 407, gap=1)
    v = _message(7)
    cg, cr = _encrypt_coeffs(g, v, 41), _encrypt_coeffs(r, v, 41)
    tg = g["bts"].trace_map(g["ev"], g["bts"].mod_raise(cg), 1, g["keys"])
    tr = r["bts"].trace_map(r["ev"], r["bts"].mod_raise(cr), 1, r["keys"])
    assert_ct_equal(tg, tr, "trace_map")
    lg, _ = g["bts"].half_bts(g["ev"], cg, g["keys"])
    lr, _ = r["bts"].half_bts(r["ev"], cr, r["keys"])
    assert_ct_equal(lg, lr, "sparse half_bts")
