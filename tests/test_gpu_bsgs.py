"""BSGS Chebyshev evaluation (BASELINE.json config 3) on the GPU against its
oracle: the same algorithm composed of the compiled reference's own Evaluator
primitives (oracle/bsgs_ref.py). Bit-exact residues and metadata, plus the
decoded values against a double Clenshaw (reference test_ckks.cpp:358-377
tolerance 2^-20) and against the reference ladder's decoded output."""
import math

import numpy as np
import pytest

from common import assert_ct_equal, dec_slots, enc_slots, make_setup
from oracle import bsgs_ref

pytestmark = pytest.mark.gpu


def clenshaw(c, x):
    b1 = b2 = 0.0
    for k in range(len(c) - 1, 0, -1):
        b1, b2 = 2 * x * b1 - b2 + c[k], b1
    return x * b1 - b2 + c[0]


@pytest.fixture(scope="module")
def pair(G, R, gpu_available):
    kw = dict(N=64, nq=10, K=2, group_size=2, seed=47)
    return make_setup(G, **kw), make_setup(R, **kw)


@pytest.fixture(params=[True, False], ids=["lazy", "eager"])
def lazy(G, request):
    """Both relinearisation orders of the BSGS tree (the product's default is
    lazy; oracle/bsgs_ref.py restates both over reference primitives)."""
    was = G.lazy_relin_enabled()
    G.set_lazy_relin(request.param)
    yield request.param
    G.set_lazy_relin(was)


@pytest.mark.parametrize("deg,odd", [(3, False), (5, True), (7, False), (15, False), (15, True), (27, True),
                                     (31, False), (63, True)])
def test_bsgs_bit_exact_vs_oracle(G, R, pair, deg, odd, lazy):
    g, r = pair
    rng = R.Rng(1000 + deg)
    coeffs = [float(int(rng.uniform(2001)) - 1000) / 4000.0 for _ in range(deg + 1)]
    if odd:
        coeffs = [0.0 if k % 2 == 0 else c for k, c in enumerate(coeffs)]
    vals = [-1.0 + (i + 0.5) / 16.0 for i in range(32)]
    cg = enc_slots(g, vals, 2.0 ** 45, G.Rng(53))
    cr = enc_slots(r, vals, 2.0 ** 45, R.Rng(53))
    og = G.eval_chebyshev_bsgs(g.ev, cg, coeffs, g.keys)
    orr = bsgs_ref.eval_chebyshev_bsgs(R, r.ev, cr, coeffs, r.keys, lazy=lazy)
    assert_ct_equal(og, orr, f"bsgs d={deg} lazy={lazy}")
    # never more levels than the reference ladder (d = 27 saves one)
    lad = R.eval_chebyshev(r.ev, cr, coeffs, r.keys)
    assert og.level() >= lad.level()
    got = dec_slots(g, og, 32).real
    for x, y in zip(vals, got):
        assert abs(y - clenshaw(coeffs, x)) < 2.0 ** -20


def test_mul2_relin_rescale_vs_reference(G, R, pair):
    """Evaluator::mul2_relin_rescale = rescale(relinearize(add(mul(a, b),
    mul(c, d)))) [+ add] over the reference's own primitives: equal and
    unequal product levels (the second tensor formed at the first's level),
    the second product BELOW the first (general path), with and without the
    addend."""
    g, r = pair
    vals = [(-1.0 + (i + 0.5) / 16.0) * 0.9 for i in range(32)]

    def mk(S, T, seed, level):
        return enc_slots(S, vals, 2.0 ** 45, T.Rng(seed), level=level)

    top = g.ring.max_level()
    for la, lb, lc, ld, ladd in [(top, top, top, top, None), (top - 2, top - 1, top, top - 1, top - 4),
                                 (top, top, top - 1, top - 2, top - 1), (top - 1, top - 1, top - 1, top, top)]:
        ag, bg, cg, dg = (mk(g, G, 60 + i, l) for i, l in enumerate((la, lb, lc, ld)))
        ar, br, cr, dr = (mk(r, R, 60 + i, l) for i, l in enumerate((la, lb, lc, ld)))
        addg = addr = None
        if ladd is not None:
            addg, addr = mk(g, G, 70, ladd), mk(r, R, 70, ladd)
        got = g.ev.mul2_relin_rescale(ag, bg, cg, dg, g.keys, addg)
        want = r.ev.rescale(r.ev.key_context().relinearize(r.ev.add(r.ev.mul(ar, br), r.ev.mul(cr, dr)),
                                                           r.keys.relin))
        if addr is not None:
            want = r.ev.add(want, addr)
        assert_ct_equal(got, want, f"mul2_relin_rescale levels {(la, lb, lc, ld, ladd)}")
        assert got.noise_bound == want.noise_bound


def test_bsgs_threshold_bit_exact(G, R, gpu_available, lazy):
    chain_g = G.build_chain(G.ThresholdParams(8, 12, [15, 15, 27], 0.0))
    chain_r = R.build_chain(R.ThresholdParams(8, 12, [15, 15, 27], 0.0))
    lv = chain_r.levels_required()
    kw = dict(N=64, nq=lv + 2, K=2, group_size=3, seed=909)
    g, r = make_setup(G, **kw), make_setup(R, **kw)
    scores = [0.1 + 0.8 * i / 31 for i in range(32)]
    d = 2.0 ** 45
    sg, tg = enc_slots(g, scores, d, G.Rng(5)), enc_slots(g, [0.5] * 32, d, G.Rng(6))
    sr, tr = enc_slots(r, scores, d, R.Rng(5)), enc_slots(r, [0.5] * 32, d, R.Rng(6))
    og = G.eval_private_threshold_plain_norm(g.ev, sg, tg, 1.0, chain_g, g.keys, G.PolyEval.bsgs)
    orr = bsgs_ref.threshold_plain_norm_bsgs(R, r.ev, sr, tr, 1.0, chain_r, r.keys, lazy=lazy)
    assert_ct_equal(og, orr, f"threshold (15,15,27) bsgs lazy={lazy}")
    bits = dec_slots(g, og, 32).real
    for s, b in zip(scores, bits):
        if abs(s - 0.5) > 2.0 ** -7:
            assert abs(b - (1.0 if s >= 0.5 else 0.0)) < 0.01
    many = G.eval_private_threshold_plain_norm_many(g.ev, [sg, sg], tg, 1.0, chain_g, g.keys, 2, G.PolyEval.bsgs)
    for o in many:
        assert_ct_equal(o, orr, "threshold bsgs (concurrent streams)")
