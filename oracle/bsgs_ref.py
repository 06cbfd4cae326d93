"""TEST INFRASTRUCTURE ONLY — the oracle for baby-step/giant-step Chebyshev
evaluation.

The reference evaluates Chebyshev series with a full T_k ladder
(eval_chebyshev, ckks.hpp:515-579); BASELINE.json config 3 asks for BSGS.
There is no reference BSGS to run, so — as SURVEY 8(c) prescribes — the
oracle is the BSGS algorithm written here ONCE over the shared Python API and
executed with the compiled, unmodified reference module (oracle/_ref): every
homomorphic step is a reference primitive (Evaluator::mul_relin, rescale,
mul_scalar, add_scalar, add; ckks.hpp:201-324). The product's C++
eval_chebyshev_bsgs performs the identical sequence; tests compare residues
bit for bit.

Algorithm (depth = ceil(log2 d) + 1, the same level budget as the ladder):
  b = 2^ceil(log2(d+1)/2) baby steps T_1..T_b and giants T_{b 2^j}, all from
  the reference's ladder recurrence T_{a+b} = 2 T_a T_b - T_{b-a} (a = k/2);
  p = q * T_n + r by Chebyshev division at the largest giant n <= deg p:
      q = [c_n, 2 c_{n+1}, ..., 2 c_m],  r_i = c_i  (i < n),  r_{n-i} -= c_{n+i};
  blocks of degree < b are the reference's combination step
      rescale( sum_k mul_scalar(T_k, c_k, s) + add_scalar(c_0) ),
  with s = q_lvl * target / scale(T_first) so that every block lands on the
  scale its consumer needs: the output at scale(x) (as the ladder's), and each
  quotient Q at target * q_lp / scale(T_n) so Q * T_n rescales onto target.
  Without this the giant-step products drift from Delta by scale(T_n)/q per
  level and deep chains (config 5, degree 63) fail the 1e-4 scale check.

Lazy relinearisation (LAZY_RELIN, the product's default): where the remainder
of a node is itself a giant-step node, p = Q T_n + (Q' T_n' + R'), the two
degree-2 products are added BEFORE relinearisation,
      rescale( relinearize( mul(Q, T_n) + mul(Q', T_n') ) ) + R',
with Q' evaluated at the scale that makes both tensors' scales equal
(target * q_lp / scale(T_n')) and the second tensor dropped to the first's
level by Evaluator::add's own level alignment: one key switch and one rescale
instead of two of each. Every step is still a reference primitive
(Evaluator::mul ckks.hpp:220-245, add :201-208, KeyContext::relinearize
rlwe.hpp:601-620, rescale ckks.hpp:315-324).
"""
from __future__ import annotations

import math
import os

# module default (the product's: TG_LAZY_RELIN=0 switches both to one key
# switch per product); eval_chebyshev_bsgs(..., lazy=...) overrides it
LAZY_RELIN = os.environ.get("TG_LAZY_RELIN", "1") != "0"


def _trim(c):
    c = list(c)
    while len(c) > 1 and c[-1] == 0.0:
        c.pop()
    return c


def eval_chebyshev_bsgs(T, ev, x, coeffs, keys, lazy=None):
    lazy = LAZY_RELIN if lazy is None else lazy
    c = _trim(coeffs)
    d = len(c) - 1
    if d == 0:
        return ev.add_scalar(ev.mul_scalar(x, 0.0, 1.0), c[0])
    if x.level() < math.ceil(math.log2(d)) + 1:
        raise RuntimeError("[ckks] insufficient levels for polynomial evaluation")
    lb = math.ceil(math.log2(d + 1) / 2)
    b = 1 << lb
    cache = {1: x}

    def get(k):  # the reference ladder step (ckks.hpp:532-555)
        if k in cache:
            return cache[k]
        a = k // 2
        bb = k - a
        ta, tb = get(a), get(bb)
        prod = ev.mul_relin(ta, tb, keys)
        prod.to_coeff()
        prod.add_inplace(prod)
        if a == bb:
            res = ev.rescale(ev.add_scalar(prod, -1.0))
        else:
            tc = get(bb - a).copy()
            tc.to_coeff()
            if tc.level() > prod.level():
                tc.drop_to_level(prod.level())
            tc = ev.mul_scalar(tc, 1.0, prod.scale / tc.scale)
            prod.sub_inplace(tc)
            res = ev.rescale(prod)
        cache[k] = res
        return res

    def base_terms(cs):
        ks = [k for k in range(1, len(cs)) if cs[k] != 0.0]
        if not ks:
            return [1], {1: 0.0}
        return ks, {k: cs[k] for k in ks}

    def level_of(cs):  # output level of rec(cs); levels do not depend on scales
        cs = _trim(cs)
        if all(v == 0.0 for v in cs):
            return None
        m = len(cs) - 1
        if m < b:
            ks_use, _ = base_terms(cs)
            return min([x.level()] + [get(k).level() for k in ks_use]) - 1
        n, q, r = split(cs)
        lq, lr = level_of(q), level_of(r)
        if lq is None:
            return lr
        lp = min(lq, get(n).level()) - 1
        return lp if lr is None else min(lp, lr)

    def base(cs, target):  # degree < b: the reference combination step (ckks.hpp:556-578)
        ks_use, cvals = base_terms(cs)
        for k in ks_use:
            get(k)
        lvl = x.level()
        for k in ks_use:
            lvl = min(lvl, get(k).level())
        # combination scale q_lvl * target / scale(T_first): the rescaled block
        # lands exactly on `target`, so giant-step products and remainders add
        # at matching scales however far the prime chain is from Delta
        comb = float(ev.ring().modulus(lvl)) * (target / get(ks_use[0]).scale)
        acc = None
        for k in ks_use:
            term = get(k).copy()
            term.to_coeff()
            if term.level() > lvl:
                term.drop_to_level(lvl)
            term = ev.mul_scalar(term, cvals[k], comb)
            if acc is None:
                acc = term
            else:
                acc.add_inplace(term)
        if cs[0] != 0.0:
            acc = ev.add_scalar(acc, cs[0])
        return ev.rescale(acc)

    def split(cs):  # Chebyshev division at the largest giant n <= deg
        m = len(cs) - 1
        n = b
        while 2 * n <= m:
            n *= 2
        q = [cs[n]] + [2.0 * cs[n + i] for i in range(1, m - n + 1)]
        r = [cs[i] for i in range(n)]
        for i in range(1, m - n + 1):
            r[n - i] = r[n - i] - cs[n + i]
        return n, q, r

    def rec(cs, target):  # the block evaluated at output scale `target`
        cs = _trim(cs)
        if all(v == 0.0 for v in cs):
            return None
        m = len(cs) - 1
        if m < b:
            return base(cs, target)
        n, q, r = split(cs)
        lq = level_of(q)
        Q = None
        if lq is not None:  # Q * T_n rescaled by q_lp must land on target
            tn = get(n)
            lp = min(lq, tn.level())
            Q = rec(q, target * float(ev.ring().modulus(lp)) / tn.scale)
            rt = _trim(r)
            if lazy and len(rt) - 1 >= b:  # the remainder is a giant-step node too
                n2, q2, r2 = split(rt)
                lq2 = level_of(q2)
                if lq2 is not None and min(lq2, get(n2).level()) >= lp:
                    tn2 = get(n2)
                    Q2 = rec(q2, target * float(ev.ring().modulus(lp)) / tn2.scale)
                    R2 = rec(r2, target)
                    both = ev.add(ev.mul(Q, tn), ev.mul(Q2, tn2))
                    P = ev.rescale(ev.key_context().relinearize(both, keys.relin))
                    return P if R2 is None else ev.add(P, R2)
        Rr = rec(r, target)
        if Q is None:
            return Rr
        P = ev.rescale(ev.mul_relin(Q, get(n), keys))
        return P if Rr is None else ev.add(P, Rr)

    out = rec(c, x.scale)
    if out is None:  # identically zero: a fresh encoding of 0 (as d == 0 does)
        return ev.add_scalar(ev.mul_scalar(x, 0.0, 1.0), 0.0)
    return out


def threshold_plain_norm_bsgs(T, ev, ct_scores, ct_t, norm, chain, keys, lazy=None):
    """eval_private_threshold_plain_norm (threshold.hpp:146-157) with every
    stage evaluated by eval_chebyshev_bsgs."""
    if ct_scores.level() < chain.levels_required():
        raise RuntimeError("[threshold] insufficient levels")
    diff = ev.sub(ct_scores, ct_t)
    diff = ev.add_scalar(diff, chain.params.epsilon / 2.0)
    ql = ev.ring().modulus(diff.level())
    u = ev.rescale(ev.mul_scalar(diff, norm, float(ql)))
    for i in range(len(chain.stages)):
        u = eval_chebyshev_bsgs(T, ev, u, chain.eval_coeffs(i), keys, lazy)
    return ev.add_scalar(u, 0.5)
