"""Hoisted rotations and the BSGS linear transform (the
CoeffToSlot/SlotToCoeff building blocks of Half-BTS) against the compiled
reference: Evaluator::apply_galois_many (ckks.hpp:338-367) and
LinearTransformPlan (ckks.hpp:373-507). Bit-exact ciphertexts; decoded
outputs against the plaintext matrix-vector product (reference tests
test_ckks.cpp mirror the same checks)."""
import numpy as np
import pytest

from common import assert_ct_equal, dec_slots, enc_slots, make_setup

pytestmark = pytest.mark.gpu


def _pair(G, R, N, n, nq=6, K=2, gs=2, seed=61):
    kw = dict(N=N, nq=nq, K=K, group_size=gs, seed=seed, q_bits=45, sp_bits=50, relin=False,
              rotations=tuple(range(1, n)), conj=True)
    return make_setup(G, **kw), make_setup(R, **kw)


def _matrix(n, seed, density=0.5):
    g = np.random.Generator(np.random.PCG64(seed))
    m = (g.uniform(-1, 1, (n, n)) + 1j * g.uniform(-1, 1, (n, n))) / n
    keep = g.random(n) < density  # drop whole diagonals: a sparse diagonal map
    keep[0] = True
    for d in range(n):
        if not keep[d]:
            for i in range(n):
                m[i][(i + d) % n] = 0
    return m


@pytest.mark.parametrize("N,n", [(64, 32), (256, 16), (1024, 512)])
def test_apply_galois_many_bit_exact(G, R, gpu_available, N, n):
    g, r = _pair(G, R, N, min(n, 32))
    vals = np.linspace(-0.7, 0.9, n)
    cg = enc_slots(g, vals, 2.0 ** 40, G.Rng(3), nslots=n)
    cr = enc_slots(r, vals, 2.0 ** 40, R.Rng(3), nslots=n)
    exps = [1] + [G.rotation_exponent(g.ring, k) for k in (1, 3, 7) if k < min(n, 32)] + [G.conjugation_exponent(g.ring)]
    og = g.ev.apply_galois_many(cg, exps, g.keys)
    orr = r.ev.apply_galois_many(cr, exps, r.keys)
    assert len(og) == len(orr) == len(exps)
    for e, a, b in zip(exps, og, orr):
        assert_ct_equal(a, b, f"hoisted exponent {e}")
    # hoisted rotation by 1 decodes to the rotated slots
    got = dec_slots(g, og[1], n).real
    assert np.max(np.abs(got - np.roll(vals, -1))) < 2.0 ** -20


@pytest.mark.parametrize("N,n,density", [(64, 32, 0.4), (64, 32, 1.0), (256, 16, 0.7)])
def test_linear_transform_bit_exact(G, R, gpu_available, N, n, density):
    g, r = _pair(G, R, N, n)
    m = _matrix(n, N + n, density)
    rows = [[complex(x) for x in row] for row in m]
    dg = G.LinearTransformPlan.diagonals_of(rows)
    dr = R.LinearTransformPlan.diagonals_of(rows)
    assert sorted(dg.keys()) == sorted(dr.keys())
    lvl = g.ring.max_level()
    pg = G.LinearTransformPlan(G.Encoder(g.ring, n), dg, float(g.ring.modulus(lvl)), lvl)
    pr = R.LinearTransformPlan(R.Encoder(r.ring, n), dr, float(r.ring.modulus(lvl)), lvl)
    assert list(pg.required_rotations()) == list(pr.required_rotations())
    assert pg.baby_count() == pr.baby_count()
    vals = np.cos(np.arange(n) * 0.37) * 0.8
    cg = enc_slots(g, vals, 2.0 ** 40, G.Rng(9), nslots=n)
    cr = enc_slots(r, vals, 2.0 ** 40, R.Rng(9), nslots=n)
    og = pg.apply(g.ev, cg, g.keys)
    orr = pr.apply(r.ev, cr, r.keys)
    assert_ct_equal(og, orr, "linear transform")
    got = dec_slots(g, og, n)
    want = m @ vals
    assert np.max(np.abs(got - want)) < 2.0 ** -20
