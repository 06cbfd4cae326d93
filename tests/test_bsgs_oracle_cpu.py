"""The BSGS oracle (oracle/bsgs_ref.py) on the CPU, over the compiled
reference: both relinearisation orders (eager: one key switch per product;
lazy: giant-step pairs added before ONE relinearisation) evaluate the same
polynomial -- decoded values against a double Clenshaw within the reference's
2^-20 tolerance (test_ckks.cpp:358-377) -- in the same level budget, and the
lazy order spends fewer key switches. No GPU needed."""
import numpy as np
import pytest

from common import dec_slots, enc_slots, load_ref, make_setup
from oracle import bsgs_ref


def clenshaw(c, x):
    b1 = b2 = 0.0
    for k in range(len(c) - 1, 0, -1):
        b1, b2 = 2 * x * b1 - b2 + c[k], b1
    return x * b1 - b2 + c[0]


class Counting:
    """Evaluator proxy counting key switches (mul_relin + relinearize)."""

    def __init__(self, ev):
        self.ev, self.ks = ev, 0
        outer = self

        class Ctx:
            def relinearize(self, ct, rlk):
                outer.ks += 1
                return ev.key_context().relinearize(ct, rlk)

        self._ctx = Ctx()

    def __getattr__(self, name):
        return getattr(self.ev, name)

    def mul_relin(self, a, b, keys):
        self.ks += 1
        return self.ev.mul_relin(a, b, keys)

    def key_context(self):
        return self._ctx


@pytest.mark.parametrize("deg,eager_ks,lazy_ks", [(15, 7, 6), (27, 10, 9), (63, 15, 13)])
def test_lazy_and_eager_orders_agree(deg, eager_ks, lazy_ks):
    R = load_ref()
    if R is None:
        pytest.skip("compiled reference oracle not built")
    S = make_setup(R, N=64, nq=10, K=2, group_size=2, seed=47)
    rng = np.random.Generator(np.random.PCG64(deg))
    coeffs = [0.0 if k % 2 == 0 else float(v) for k, v in enumerate(rng.uniform(-0.25, 0.25, deg + 1))]
    vals = np.linspace(-0.95, 0.95, 32)
    ct = enc_slots(S, vals, 2.0 ** 45, R.Rng(11))
    out = {}
    for lazy in (False, True):
        ev = Counting(S.ev)
        res = bsgs_ref.eval_chebyshev_bsgs(R, ev, ct, coeffs, S.keys, lazy=lazy)
        got = dec_slots(S, res, 32).real
        for x, y in zip(vals, got):
            assert abs(y - clenshaw(coeffs, x)) < 2.0 ** -20
        out[lazy] = (res.level(), ev.ks)
    assert out[True][0] == out[False][0]  # the same level budget
    assert out[False][1] == eager_ks and out[True][1] == lazy_ks
