"""Fused key-switch core (tg_ks_fused.cuh) vs the compiled reference.

Rings whose moduli all take the FP64 path (50-bit q-chain AND 50-bit special
primes, the configs 3-5 parameters) with N in the warp-NTT range 2^14..2^16
run key switching through kw_ks_chunks: digits' forward chunk phase, key
inner product (KeyContext::ks_inner, rlwe.hpp:501-540) and the accumulators'
inverse chunk phase in one pass. Relinearisation (rlwe.hpp:601-620), Galois
key switching (rlwe.hpp:637-654) and batched relinearisation must stay bit-
exact with the reference at full and partial digit counts.
"""
from __future__ import annotations

import pytest

from common import assert_ct_equal, make_setup

pytestmark = pytest.mark.gpu


def _cts(S, n, level, seed):
    T = S.T
    rng = T.Rng(seed)
    out = []
    for i in range(n):
        c = T.Ciphertext()
        c.parts = [T.sample_uniform(S.ring, level, 0, rng.split(10 * i + j)) for j in range(2)]
        c.scale = 2.0 ** 50
        c.domain = T.Domain.slots
        c.sk_id = S.sk.id()
        out.append(c)
    return out


@pytest.mark.parametrize("N,nq,K,gs,sp_bits", [(1 << 14, 9, 4, 3, 50), (1 << 15, 8, 3, 3, 50), (1 << 16, 7, 3, 3, 50),
                                                (1 << 14, 8, 2, 2, 60), (1 << 15, 7, 3, 3, 60), (1 << 16, 6, 2, 3, 60)])
def test_fused_keyswitch_bit_exact(G, R, gpu_available, N, nq, K, gs, sp_bits):
    """sp_bits 60: mixed rings (config 1's shape) -- FP64 q-chain rows in
    kw_ks_chunks, the 60-bit special rows in kw_ks_chunks_int."""
    kw = dict(N=N, nq=nq, K=K, group_size=gs, seed=11, q_bits=50, sp_bits=sp_bits, h=192, rotations=(1, 5))
    g, r = make_setup(G, **kw), make_setup(R, **kw)
    top = g.ring.max_level()
    for level in (top, 4, 2):  # full, partial (own row in the last digit) and small digit counts
        (a_g, b_g), (a_r, b_r) = _cts(g, 2, level, 100 + level), _cts(r, 2, level, 100 + level)
        assert_ct_equal(g.ev.mul_relin(a_g, b_g, g.keys), r.ev.mul_relin(a_r, b_r, r.keys),
                        f"mul_relin N={N} level={level}")
        assert_ct_equal(g.ev.mul_relin(a_g, a_g, g.keys), r.ev.mul_relin(a_r, a_r, r.keys),
                        f"square N={N} level={level}")
        for k in (1, 5):
            assert_ct_equal(g.ev.rotate(a_g, k, g.keys), r.ev.rotate(a_r, k, r.keys),
                            f"rotate {k} N={N} level={level}")


@pytest.mark.parametrize("batch,sp_bits", [(3, 50), (8, 50), (8, 60)])
def test_fused_keyswitch_batched(G, R, gpu_available, batch, sp_bits):
    kw = dict(N=1 << 14, nq=8, K=3, group_size=3, seed=13, q_bits=50, sp_bits=sp_bits, h=192)
    g, r = make_setup(G, **kw), make_setup(R, **kw)
    level = g.ring.max_level()
    xs_g, ys_g = _cts(g, batch, level, 7), _cts(g, batch, level, 8)
    xs_r, ys_r = _cts(r, batch, level, 7), _cts(r, batch, level, 8)
    prod = g.ev.rescale(g.ev.mul_relin(G.stack_ciphertexts(xs_g), G.stack_ciphertexts(ys_g), g.keys))
    for i, got in enumerate(G.unstack_ciphertext(prod)):
        assert_ct_equal(got, r.ev.rescale(r.ev.mul_relin(xs_r[i], ys_r[i], r.keys)), f"batched relin block {i}")


@pytest.mark.parametrize("N", [1 << 12, 1 << 16])
def test_rescale_add_matches_add_of_rescale(G, R, gpu_available, N):
    """Evaluator::rescale_add (one pass) == add(rescale(prod), y) of the
    reference, for y at a lower / equal / higher level, a level-dropped view,
    an eval-form y (two-op fallback) and a batch."""
    kw = dict(N=N, nq=7, K=3, group_size=3, seed=17, q_bits=50, sp_bits=50, h=192)
    g, r = make_setup(G, **kw), make_setup(R, **kw)
    top = g.ring.max_level()
    (a_g, b_g), (a_r, b_r) = _cts(g, 2, top, 5), _cts(r, 2, top, 5)
    prod_g, prod_r = g.ev.mul_relin(a_g, b_g, g.keys), r.ev.mul_relin(a_r, b_r, r.keys)
    for ylvl in (top - 3, top - 1, top):
        (y_g,), (y_r,) = _cts(g, 1, ylvl, 9 + ylvl), _cts(r, 1, ylvl, 9 + ylvl)
        want = r.ev.add(r.ev.rescale(prod_r), y_r)
        assert_ct_equal(g.ev.rescale_add(prod_g, y_g), want, f"rescale_add y level {ylvl}")
    (y_g,), (y_r,) = _cts(g, 1, top, 21), _cts(r, 1, top, 21)
    yv = y_g.copy()
    yv.drop_to_level(top - 2)  # a level-dropped view (strided parts)
    yr = y_r.copy()
    yr.drop_to_level(top - 2)
    assert_ct_equal(g.ev.rescale_add(prod_g, yv), r.ev.add(r.ev.rescale(prod_r), yr), "rescale_add view")
    ye = y_g.copy()
    ye.to_eval()  # fallback path
    yre = y_r.copy()
    yre.to_eval()
    assert_ct_equal(g.ev.rescale_add(prod_g, ye), r.ev.add(r.ev.rescale(prod_r), yre), "rescale_add eval y")
    xs_g, ys_g = _cts(g, 3, top, 31), _cts(g, 3, top - 1, 32)
    xs_r, ys_r = _cts(r, 3, top, 31), _cts(r, 3, top - 1, 32)
    pb = g.ev.mul_relin(G.stack_ciphertexts(xs_g), G.stack_ciphertexts(xs_g), g.keys)
    got = G.unstack_ciphertext(g.ev.rescale_add(pb, G.stack_ciphertexts(ys_g)))
    for i in range(3):
        want = r.ev.add(r.ev.rescale(r.ev.mul_relin(xs_r[i], xs_r[i], r.keys)), ys_r[i])
        assert_ct_equal(got[i], want, f"rescale_add batch block {i}")


@pytest.mark.parametrize("N,batch", [(1 << 14, 8), (1 << 16, 1), (1 << 16, 8)])
def test_mul_relin_rescale_matches_reference(G, R, gpu_available, N, batch):
    """Evaluator::mul_relin_rescale (ModDown + rescale_round (+ add) in one
    pass, tg_relinearize_tensor_rescale_batch) == rescale(mul_relin) and
    add(rescale(mul_relin), y) of the reference: residues, scale and noise
    bound. Batches that fill the GPU take the fused ModDown (N=2^16 x 8,
    2^14 x 8), a single 2^16 product the relinearise-then-rescale fallback;
    y at lower / equal level, a level-dropped view and an eval-form y."""
    kw = dict(N=N, nq=7, K=3, group_size=3, seed=19, q_bits=50, sp_bits=50, h=192)
    g, r = make_setup(G, **kw), make_setup(R, **kw)
    top = g.ring.max_level()

    def stack(T, cts):
        return cts[0] if len(cts) == 1 else T.stack_ciphertexts(cts)

    def unstack(T, ct):
        return T.unstack_ciphertext(ct) if ct.batch > 1 else [ct]

    for level in (top, 3):
        xs_g, ys_g = _cts(g, batch, level, 41 + level), _cts(g, batch, level, 42 + level)
        xs_r, ys_r = _cts(r, batch, level, 41 + level), _cts(r, batch, level, 42 + level)
        got = g.ev.mul_relin_rescale(stack(G, xs_g), stack(G, ys_g), g.keys)
        two = g.ev.rescale(g.ev.mul_relin(stack(G, xs_g), stack(G, ys_g), g.keys))
        assert got.noise_bound == two.noise_bound
        for i, c in enumerate(unstack(G, got)):
            want = r.ev.rescale(r.ev.mul_relin(xs_r[i], ys_r[i], r.keys))
            assert_ct_equal(c, want, f"mul_relin_rescale level {level} block {i}")
            assert c.noise_bound == want.noise_bound
        for ylvl in sorted({level - 2, level - 1}):
            if ylvl < 0:
                continue
            ad_g, ad_r = _cts(g, batch, ylvl, 50 + ylvl), _cts(r, batch, ylvl, 50 + ylvl)
            got = g.ev.mul_relin_rescale(stack(G, xs_g), stack(G, ys_g), g.keys, stack(G, ad_g))
            for i, c in enumerate(unstack(G, got)):
                want = r.ev.add(r.ev.rescale(r.ev.mul_relin(xs_r[i], ys_r[i], r.keys)), ad_r[i])
                assert_ct_equal(c, want, f"mul_relin_rescale add level {level} y {ylvl} block {i}")
                assert c.noise_bound == want.noise_bound
    # a level-dropped view of y (strided parts) and an eval-form y (two-op path)
    xs_g, ys_g = _cts(g, batch, top, 61), _cts(g, batch, top, 62)
    xs_r, ys_r = _cts(r, batch, top, 61), _cts(r, batch, top, 62)
    ad_g, ad_r = _cts(g, batch, top, 63), _cts(r, batch, top, 63)
    yv = stack(G, ad_g).copy()
    yv.drop_to_level(top - 2)
    ye = stack(G, ad_g).copy()
    ye.to_eval()
    for y, what in ((yv, "view"), (ye, "eval y")):
        got = unstack(G, g.ev.mul_relin_rescale(stack(G, xs_g), stack(G, ys_g), g.keys, y))
        for i, c in enumerate(got):
            yr = ad_r[i].copy()
            if what == "view":
                yr.drop_to_level(top - 2)
            else:
                yr.to_eval()
            want = r.ev.add(r.ev.rescale(r.ev.mul_relin(xs_r[i], ys_r[i], r.keys)), yr)
            assert_ct_equal(c, want, f"mul_relin_rescale {what} block {i}")


@pytest.mark.parametrize("N,batch", [(1 << 16, 8), (1 << 14, 3), (1 << 16, 1)])
def test_mul2_relin_rescale_matches_reference(G, R, gpu_available, N, batch):
    """Evaluator::mul2_relin_rescale (lazy relinearisation of a giant-step
    pair) on the fused key-switch path and as ciphertext batches:
    rescale(relinearize(add(mul(a, b), mul(c, d)))) [+ add] of the reference
    (ckks.hpp:220-245, :201-208, rlwe.hpp:601-620, ckks.hpp:315-324), with
    the second product above the first's level (level-dropped operand views)
    and at it."""
    kw = dict(N=N, nq=7, K=3, group_size=3, seed=23, q_bits=50, sp_bits=50, h=192)
    g, r = make_setup(G, **kw), make_setup(R, **kw)
    top = g.ring.max_level()

    def stack(T, cts):
        return cts[0] if len(cts) == 1 else T.stack_ciphertexts(cts)

    def unstack(T, ct):
        return T.unstack_ciphertext(ct) if ct.batch > 1 else [ct]

    for (la, lc, ld, ladd) in [(top - 1, top, top - 1, top - 3), (top, top, top, None), (3, 5, 4, 2)]:
        lv = (la, la, lc, ld)
        ops_g = [_cts(g, batch, l, 80 + 7 * i + l) for i, l in enumerate(lv)]
        ops_r = [_cts(r, batch, l, 80 + 7 * i + l) for i, l in enumerate(lv)]
        ad_g = ad_r = None
        if ladd is not None:
            ad_g, ad_r = _cts(g, batch, ladd, 99), _cts(r, batch, ladd, 99)
        got = g.ev.mul2_relin_rescale(*(stack(G, o) for o in ops_g), g.keys, stack(G, ad_g) if ad_g else None)
        for i, c in enumerate(unstack(G, got)):
            a, b, cc, d = (o[i] for o in ops_r)
            want = r.ev.rescale(r.ev.key_context().relinearize(r.ev.add(r.ev.mul(a, b), r.ev.mul(cc, d)),
                                                               r.keys.relin))
            if ad_r:
                want = r.ev.add(want, ad_r[i])
            assert_ct_equal(c, want, f"mul2_relin_rescale N={N} levels {lv} block {i}")
            assert c.noise_bound == want.noise_bound


@pytest.mark.parametrize("N,batch", [(1 << 16, 3), (1 << 14, 2), (1 << 14, 8)])
def test_ladder_step_in_moddown_matches_reference(G, R, gpu_available, N, batch):
    """The Chebyshev ladder (ckks.hpp:532-555) with each step's linear part
    and rescale applied inside the product's ModDown
    (tg_relinearize_tensor_ladder_batch: N=2^16 x 3 and 2^14 x 8 fill the GPU
    and take the fused pass, 2^14 x 2 the relinearise-then-lincomb fallback):
    eval_chebyshev of degree 6 (T_2 = 2 T_1^2 - 1, T_3 = 2 T_1 T_2 - T_1 with a
    level-dropped T_1, T_4, T_5, T_6) on a ciphertext batch vs the unmodified
    reference per block, residues and metadata."""
    kw = dict(N=N, nq=7, K=3, group_size=3, seed=29, q_bits=50, sp_bits=50, h=192)
    g, r = make_setup(G, **kw), make_setup(R, **kw)
    from common import enc_slots
    import numpy as np
    coeffs = [0.11, -0.32, 0.27, 0.19, -0.08, 0.21, -0.13]
    vals = [np.linspace(-0.9, 0.9, 64) * (1.0 - 0.1 * i) for i in range(batch)]
    cg = [enc_slots(g, v, 2.0 ** 50, G.Rng(70 + i)) for i, v in enumerate(vals)]
    cr = [enc_slots(r, v, 2.0 ** 50, R.Rng(70 + i)) for i, v in enumerate(vals)]
    got = G.eval_chebyshev(g.ev, G.stack_ciphertexts(cg) if batch > 1 else cg[0], coeffs, g.keys)
    for i, c in enumerate(G.unstack_ciphertext(got) if batch > 1 else [got]):
        want = R.eval_chebyshev(r.ev, cr[i], coeffs, r.keys)
        assert_ct_equal(c, want, f"ladder N={N} block {i}")
        assert c.noise_bound == want.noise_bound
