"""Eval-form pipeline: the
products, combinations and rescales of the Chebyshev evaluators stay in
evaluation form. Each eval-form primitive, transformed back to coefficient
form, must equal its coefficient-form counterpart residue for residue (which
the other suites pin to the compiled reference), and the evaluators must give
identical ciphertexts with the pipeline on and off and against the reference
ladder / the BSGS oracle."""
import numpy as np
import pytest

from common import assert_ct_equal, enc_slots, make_setup
from oracle import bsgs_ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setups(G, R, gpu_available):
    kw = dict(N=256, nq=8, K=3, group_size=3, seed=71)
    return make_setup(G, **kw), make_setup(R, **kw)


def _coeff(ct):
    c = ct
    c.to_coeff()
    return c


@pytest.mark.parametrize("batch", [1, 3])
def test_relinearize_and_rescale_eval(G, setups, batch):
    g, _ = setups
    vals = np.linspace(-0.9, 0.8, 64)
    xs = [enc_slots(g, vals * (i + 1) / 4, 2.0 ** 40, G.Rng(10 + i)) for i in range(batch)]
    ys = [enc_slots(g, vals[::-1], 2.0 ** 40, G.Rng(20 + i)) for i in range(batch)]
    x = G.stack_ciphertexts(xs) if batch > 1 else xs[0]
    y = G.stack_ciphertexts(ys) if batch > 1 else ys[0]
    want = g.ev.mul_relin(x, y, g.keys)
    got = g.ev.mul_relin_eval(x, y, g.keys)
    assert int(got.form()) != int(want.form())  # stays in eval form
    want_c = _coeff(want)
    assert_ct_equal(_coeff(got), want_c, f"relinearize_eval B={batch}")
    # rescale on eval-form input, eval-form output
    e = g.ev.mul_relin_eval(x, y, g.keys)
    rs = g.ev.rescale_eval(e)
    assert rs.level() == want_c.level() - 1
    assert_ct_equal(_coeff(rs), g.ev.rescale(want_c), f"rescale_eval B={batch}")


def test_rescale_eval_level_dropped_and_low_level(G, setups):
    g, _ = setups
    vals = np.linspace(-0.5, 0.5, 64)
    c = enc_slots(g, vals, 2.0 ** 40, G.Rng(3))
    for lvl in (5, 1):
        d = g.ev.mul_scalar(c, 0.75, 1.0)
        d.drop_to_level(lvl)  # a level-dropped view: per-poly launches
        want = g.ev.rescale(d)
        e = d
        e.to_eval()
        assert_ct_equal(_coeff(g.ev.rescale_eval(e)), want, f"rescale_eval level {lvl}")


@pytest.mark.parametrize("deg", [7, 15, 27])
def test_chebyshev_pipelines_identical(G, R, setups, deg):
    g, r = setups
    rng = np.random.Generator(np.random.PCG64(deg))
    coeffs = [float(v) for v in rng.uniform(-0.5, 0.5, deg + 1)]
    vals = np.linspace(-0.95, 0.95, 64)
    cg = enc_slots(g, vals, 2.0 ** 45, G.Rng(9))
    cr = enc_slots(r, vals, 2.0 ** 45, R.Rng(9))
    was, was_lazy = G.eval_pipeline_enabled(), G.lazy_relin_enabled()
    try:
        out = {}
        G.set_lazy_relin(False)  # the eval-form pipeline relinearises every product
        for on in (True, False):
            G.set_eval_pipeline(on)
            out[on] = (G.eval_chebyshev(g.ev, cg, coeffs, g.keys), G.eval_chebyshev_bsgs(g.ev, cg, coeffs, g.keys))
    finally:
        G.set_eval_pipeline(was)
        G.set_lazy_relin(was_lazy)
    assert_ct_equal(out[True][0], out[False][0], f"ladder on/off d={deg}")
    assert_ct_equal(out[True][1], out[False][1], f"bsgs on/off d={deg}")
    assert_ct_equal(out[True][0], R.eval_chebyshev(r.ev, cr, coeffs, r.keys), f"ladder vs reference d={deg}")
    assert_ct_equal(out[True][1], bsgs_ref.eval_chebyshev_bsgs(R, r.ev, cr, coeffs, r.keys, lazy=False),
                    f"bsgs vs oracle d={deg}")
    # the result's eval form is cached: the next product does not re-transform it
    nxt = g.ev.mul_relin(out[True][0], out[True][0], g.keys)
    assert nxt.level() == out[True][0].level()


@pytest.mark.parametrize("batch", [1, 2])
def test_eval_pipeline_warp_ntt_n65536(G, gpu_available, batch):
    """The same identities at N = 2^16 with 50-bit q-chain AND special primes:
    the warp NTT kernels with row ranges (rescale_eval's single inverse row
    and per-modulus forward rows) on the column-pair path, and the fused
    key-switch core in the coefficient-form reference products."""
    g = make_setup(G, N=1 << 16, nq=6, K=3, group_size=3, seed=73, q_bits=50, sp_bits=50, h=192)
    vals = np.linspace(-0.9, 0.8, 64)
    xs = [enc_slots(g, vals * (i + 1) / 4, 2.0 ** 45, G.Rng(30 + i)) for i in range(batch)]
    ys = [enc_slots(g, vals[::-1], 2.0 ** 45, G.Rng(40 + i)) for i in range(batch)]
    x = G.stack_ciphertexts(xs) if batch > 1 else xs[0]
    y = G.stack_ciphertexts(ys) if batch > 1 else ys[0]
    want_c = _coeff(g.ev.mul_relin(x, y, g.keys))
    assert_ct_equal(_coeff(g.ev.mul_relin_eval(x, y, g.keys)), want_c, f"relinearize_eval N=2^16 B={batch}")
    rs = g.ev.rescale_eval(g.ev.mul_relin_eval(x, y, g.keys))
    assert_ct_equal(_coeff(rs), g.ev.rescale(want_c), f"rescale_eval N=2^16 B={batch}")
