"""Composed query paths on the device vs the reference:
config 2's encrypted linear score (8 pt x ct MACs + rescale) at full size,
and the full TETRIS statement of configs 4/5 (three private thresholds, AND,
plaintext flag, slot-sum) at reduced N with the configs' own level chains,
gadgets and minimax degrees. Ladder mode is compared with the unmodified
reference; BSGS mode with its restatement over reference primitives
(oracle/bsgs_ref.py). Bit-exact ciphertexts, exact decrypted counts."""
import dataclasses

import numpy as np
import pytest

from common import assert_ct_equal, copy_chain, mirror_encoder
from oracle import bsgs_ref
from paper_2412_13269_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _decode(S, ct):
    m = S.ctx.decrypt(S.sk, ct)
    return np.array(S.T.Encoder(S.ring, S.spec.slots).decode_slots(m, ct.scale))


def test_config2_linear_score_full_size(G, R, gpu_available):
    spec = dataclasses.replace(W.CONFIGS[2], records=1 << 15, n_cts=2)
    g, r = W.make_context(G, spec, relin=False), W.make_context(R, spec, relin=False)
    r.encode = mirror_encoder(g, R)
    attrs, w = W.linear_score_data(spec)
    ig, ir = W.config2_inputs(g, attrs, w), W.config2_inputs(r, attrs, w)
    sg = W.config2_query(g, ig, streams=2)
    sr = W.config2_query(r, ir)
    n = spec.slots
    for b in range(spec.n_cts):
        assert_ct_equal(sg[b], sr[b], f"linear score block {b}")
        got = _decode(g, sg[b]).real
        want = attrs[b * n:(b + 1) * n] @ w / W.ATTR_NORM
        assert np.max(np.abs(got - want)) < 2.0 ** -20


def _statement(G, R, spec, chain_g, t_override=None):
    rot = W.inner_sum_rotations(spec.slots)
    g, r = W.make_context(G, spec, rotations=rot), W.make_context(R, spec, rotations=rot)
    r.encode = mirror_encoder(g, R)
    chain_r = copy_chain(R, chain_g)
    d = W.statement_data(spec)
    if t_override:
        d.t = t_override
    qg, qr = W.statement_query_inputs(g, d), W.statement_query_inputs(r, d)
    bg = [W.statement_block_inputs(g, d, b) for b in range(spec.n_cts)]
    br = [W.statement_block_inputs(r, d, b) for b in range(spec.n_cts)]
    return g, r, chain_r, d, qg, qr, bg, br


@pytest.fixture(scope="module")
def stmt4(G, R, gpu_available):
    spec = dataclasses.replace(W.CONFIGS[4], N=1024, records=2048, n_cts=4)
    chain = W.config3_chain(G, spec)
    # looser thresholds than the config's clinical ones so that a 2^11-record
    # sample has a non-trivial count
    return (spec, chain) + _statement(G, R, spec, chain, t_override=(0.2, 0.3, -0.02))


def test_config4_statement_ladder_bit_exact(G, R, stmt4):
    spec, chain_g, g, r, chain_r, d, qg, qr, bg, br = stmt4
    acc_g = W.statement_partial(g, qg, bg, W.threshold_fn(g, chain_g, G.PolyEval.ladder), streams=3)
    acc_r = W.statement_partial(r, qr, br, W.threshold_fn(r, chain_r))
    assert acc_g.level() == 1
    assert_ct_equal(acc_g, acc_r, "statement partial (ladder)")
    cg = G.inner_sum(g.ev, acc_g, spec.slots, g.keys)
    cr = R.inner_sum(r.ev, acc_r, spec.slots, r.keys)
    assert_ct_equal(cg, cr, "statement count (ladder)")
    count_g, count_r = _decode(g, cg)[0].real, _decode(r, cr)[0].real
    assert round(count_g) == round(count_r)
    plain = W.statement_plain_count(d)
    assert abs(count_g - plain) < 3, (count_g, plain)  # slots inside the 2^-alpha gap may be fractional


def test_config4_statement_bsgs_bit_exact(G, R, stmt4):
    spec, chain_g, g, r, chain_r, d, qg, qr, bg, br = stmt4
    acc_g = W.statement_partial(g, qg, bg, W.threshold_fn(g, chain_g, G.PolyEval.bsgs), streams=4)

    def thr_r(x, t, norm):
        return bsgs_ref.threshold_plain_norm_bsgs(R, r.ev, x, t, norm, chain_r, r.keys)

    acc_r = W.statement_partial(r, qr, br, thr_r)
    assert_ct_equal(acc_g, acc_r, "statement partial (bsgs)")
    per_slot = _decode(g, acc_g).real
    assert abs(per_slot.sum() - W.statement_plain_count(d)) < 3


def test_config4_statement_batched_bit_exact(G, R, stmt4):
    """Blocks evaluated as ciphertext batches (one batched threshold per
    column group, batched AND products) == the reference per block."""
    spec, chain_g, g, r, chain_r, d, qg, qr, bg, br = stmt4
    for mode, thr_r in ((G.PolyEval.ladder, W.threshold_fn(r, chain_r)),
                        (G.PolyEval.bsgs,
                         lambda x, t, norm: bsgs_ref.threshold_plain_norm_bsgs(R, r.ev, x, t, norm, chain_r, r.keys))):
        acc_g = W.statement_partial_batched(g, qg, bg, W.threshold_fn(g, chain_g, mode), streams=2, max_blocks=3)
        acc_r = W.statement_partial(r, qr, br, thr_r)
        assert acc_g.batch == 1
        assert_ct_equal(acc_g, acc_r, f"batched statement ({mode})")


def test_batch_ops_match_single(G, gpu_available):
    """stack / slice / unstack round trip and batch-aware ops (tensor,
    relinearize, add_scalar, fused combinations) against single ciphertexts."""
    spec = dataclasses.replace(W.CONFIGS[4], N=256, nq=6, K=2, group=2, records=512, n_cts=4)
    g = W.make_context(G, spec)
    vals = [np.linspace(-0.5, 0.5, spec.slots) * (i + 1) / 4 for i in range(3)]
    cts = W.encrypt_many(g, vals, g.ring.max_level(), [1, 2, 3])
    fat = G.stack_ciphertexts(cts)
    assert fat.batch == 3 and fat.degree() == 1
    for a, b in zip(G.unstack_ciphertext(fat), cts):
        assert_ct_equal(a, b, "unstack")
    prod = g.ev.rescale(g.ev.mul_relin(fat, fat, g.keys))
    sq = [g.ev.rescale(g.ev.mul_relin(c, c, g.keys)) for c in cts]
    for a, b in zip(G.unstack_ciphertext(prod), sq):
        assert_ct_equal(a, b, "batched mul_relin + rescale")
    sc = g.ev.add_scalar(prod, 0.25)
    for a, b in zip(G.unstack_ciphertext(sc), sq):
        assert_ct_equal(a, g.ev.add_scalar(b, 0.25), "batched add_scalar")
    mid = G.slice_ciphertext(prod, 1, 2)
    for a, b in zip(G.unstack_ciphertext(g.ev.add(mid, mid)), sq[1:]):
        assert_ct_equal(a, g.ev.add(b, b), "slice + add")
    coeffs = [0.1, 0.5, 0.0, -0.25]
    ch = G.eval_chebyshev(g.ev, fat, coeffs, g.keys)
    for a, b in zip(G.unstack_ciphertext(ch), cts):
        assert_ct_equal(a, G.eval_chebyshev(g.ev, b, coeffs, g.keys), "batched eval_chebyshev")


def test_config5_statement_deg63_bsgs_bit_exact(G, R, gpu_available):
    """Config 5's chain (three degree-63 stages, alpha 13), L = 28, dnum = 3
    (group 10 under 9 special primes) at N = 1024."""
    spec = dataclasses.replace(W.CONFIGS[5], N=1024, records=1024, n_cts=2)
    chain_g = W.config3_chain(G, spec)
    assert chain_g.levels_required() == 22
    g, r, chain_r, d, qg, qr, bg, br = _statement(G, R, spec, chain_g, t_override=(0.2, 0.3, -0.02))
    acc_g = W.statement_partial(g, qg, bg, W.threshold_fn(g, chain_g, G.PolyEval.bsgs), streams=2)

    def thr_r(x, t, norm):
        return bsgs_ref.threshold_plain_norm_bsgs(R, r.ev, x, t, norm, chain_r, r.keys)

    acc_r = W.statement_partial(r, qr, br, thr_r)
    assert_ct_equal(acc_g, acc_r, "config-5 statement partial (bsgs)")
    assert acc_g.level() >= 3
    per_slot = _decode(g, acc_g).real
    assert abs(per_slot.sum() - W.statement_plain_count(d)) < 3
