"""TEST INFRASTRUCTURE ONLY — full-size parity of the shipped path.

The path bench.py times (BSGS polynomial evaluation, record blocks stacked as
ciphertext batches, N = 2^16 with the configs' own chains and gadgets) is
checked against the BSGS oracle: oracle/bsgs_ref.py executing every
homomorphic step with the compiled, unmodified reference (oracle/_ref), on the
same seeded inputs (keys and encryptions bit-identical, slot vectors encoded
once on the device, whose encoder is bit-identical to the reference's —
tests/test_gpu_encoder.py). Used by tests/test_gpu_fullsize.py and by
bench.py's cpu_baseline leg (the checker there, after the timed region).

Reference order: threshold per (block, column) (threshold.hpp:146-157 with
eval_chebyshev's BSGS restatement), AND as rescale(mul_relin(b1, b2)) then
x b3, the plaintext flag, sum over blocks, one inner_sum
(protocol.hpp:319-323, ckks.hpp:605-615).
"""
from __future__ import annotations

import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from common import copy_chain, mirror_encoder
from oracle import bsgs_ref


def oracle_context(R, W, spec, S_gpu, chain_gpu, rotations=True):
    """Reference context with the workload's keys (same seeds as the device
    context), the device encoder feeding it residues, and the same chain."""
    rot = W.inner_sum_rotations(spec.slots) if rotations else []
    SR = W.make_context(R, spec, rotations=rot, relin=bool(spec.degrees))
    SR.encode = mirror_encoder(S_gpu, R)
    chain = copy_chain(R, chain_gpu) if chain_gpu is not None else None
    return SR, chain


def oracle_threshold(R, SR, chain):
    def thr(x, t, norm):
        return bsgs_ref.threshold_plain_norm_bsgs(R, SR.ev, x, t, norm, chain, SR.keys)
    return thr


def oracle_statement_blocks(R, W, SR, chain, d, block_ids, threads):
    """Per-block statement outputs (before the sum) through the BSGS oracle:
    every (block, column) threshold on a thread pool, then each block's AND
    and flag product in statement_block's order. Returns (outs, seconds of
    the evaluation, excluding input preparation)."""
    q = W.statement_query_inputs(SR, d)
    blocks = [W.statement_block_inputs(SR, d, b) for b in block_ids]
    thr = oracle_threshold(R, SR, chain)
    ev, keys = SR.ev, SR.keys
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max(1, threads)) as ex:
        risks = list(ex.map(lambda b: W.linear_score(SR, q.ct_w, b.pt_attr, b.attr_scale), blocks))
        futs = [(ex.submit(thr, b.ct_sugar, q.ct_t[0], 1.0), ex.submit(thr, b.ct_bp, q.ct_t[1], 1.0),
                 ex.submit(thr, r, q.ct_t[2], W.RISK_NORM)) for b, r in zip(blocks, risks)]

        def finish(i):
            b, (f1, f2, f3) = blocks[i], futs[i]
            a = ev.rescale(ev.mul_relin(f1.result(), f2.result(), keys))
            a = ev.rescale(ev.mul_relin(a, f3.result(), keys))
            return ev.rescale(ev.mul_plain(a, b.pt_flag, b.flag_scale))

        outs = list(ex.map(finish, range(len(blocks))))
    return outs, time.perf_counter() - t0


def oracle_threshold_count(R, W, SR, chain, scores, thr_value, block_ids, threads):
    """Config 3 through the BSGS oracle: threshold of every score block (one
    thread each), sum in block order, one inner_sum. Returns (count ct,
    per-block outputs, seconds)."""
    spec = SR.spec
    n, L = spec.slots, SR.ring.max_level()
    cts = W.encrypt_many(SR, [scores[b * n:(b + 1) * n] for b in block_ids], L, [100 + b for b in block_ids])
    ct_t = W.encrypt_many(SR, [[thr_value] * n], L, [99])[0]
    thr = oracle_threshold(R, SR, chain)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max(1, threads)) as ex:
        outs = list(ex.map(lambda c: thr(c, ct_t, spec.norm), cts))
    acc = outs[0]
    for o in outs[1:]:
        acc = SR.ev.add(acc, o)
    count = R.inner_sum(SR.ev, acc, spec.slots, SR.keys)
    return count, outs, time.perf_counter() - t0


def ct_equal(a, b) -> bool:
    """Bit-exact ciphertext equality (residues, level, scale, degree)."""
    return (a.level() == b.level() and a.scale == b.scale and len(a.parts) == len(b.parts)
            and all(np.array_equal(x.to_numpy(), y.to_numpy()) for x, y in zip(a.parts, b.parts)))


def decrypted_count(S, ct) -> float:
    enc = S.T.Encoder(S.ring, S.spec.slots)
    return float(np.array(enc.decode_slots(S.ctx.decrypt(S.sk, ct), ct.scale))[0].real)


def sum_and_count(S, outs):
    """inner_sum of the mod-q sum of `outs` (block order) in S's module."""
    acc = outs[0]
    for o in outs[1:]:
        acc = S.ev.add(acc, o)
    return S.T.inner_sum(S.ev, acc, S.spec.slots, S.keys)
