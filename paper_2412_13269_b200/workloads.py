"""BASELINE.json workloads (configs 1-5), written once against the shared
Python API so the same code drives the B200 module and the compiled reference
(oracle/_ref, test/bench checker only).

Synthetic data (there is no dataset): every record attribute is drawn from a
seeded numpy PCG64 stream with BASELINE.json's distributions; the reference's
own Rng drives keys, noise and encryption randomness. Parameter choices left
open by BASELINE.json are fixed here and documented in DESIGN.md.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from types import SimpleNamespace

import numpy as np


@dataclass(frozen=True)
class Spec:
    name: str
    N: int
    nq: int                 # q-chain length (max_level + 1)
    q_bits: int             # arithmetic primes (~= log2 Delta)
    K: int                  # special primes
    sp_bits: int
    group: int              # gadget group size (dnum = ceil(nq / group))
    h: int                  # secret Hamming weight
    delta_log2: int
    q0_bits: int | None = None
    degrees: tuple = ()
    alpha: int = 8
    beta: int = 12
    epsilon: float = 0.0
    norm: float = 1.0
    n_cts: int = 1
    records: int = 0
    seed: int = 0x7e7215

    @property
    def slots(self) -> int:
        return self.N // 2

    @property
    def delta(self) -> float:
        return float(2 ** self.delta_log2)


CONFIGS = {
    # configs[0]: ring-op microbench, 64 ciphertexts of uniform residues
    1: Spec("config1-ringops", N=1 << 14, nq=8, q_bits=50, K=2, sp_bits=60, group=2, h=192, delta_log2=50,
            n_cts=64, records=0, seed=0xC0F1),
    # configs[1]: encrypted linear score, 2^16 records x 8 attributes
    2: Spec("config2-linear-score", N=1 << 15, nq=4, q_bits=40, q0_bits=60, K=1, sp_bits=60, group=4, h=192,
            delta_log2=40, n_cts=4, records=1 << 16, seed=0xC0F2),
    # configs[2]: private threshold count, 2^17 records, (15,15,27)
    3: Spec("config3-threshold-count", N=1 << 16, nq=21, q_bits=50, K=6, sp_bits=60, group=7, h=192,
            delta_log2=50, degrees=(15, 15, 27), alpha=8, epsilon=0.0, norm=1.0, n_cts=4, records=1 << 17,
            seed=0xC0F3),
}


def _primes(T, spec: Spec):
    two_n = 2 * spec.N
    if spec.q0_bits:
        q0 = list(T.find_ntt_primes(spec.q0_bits, 1, two_n))
        qs = q0 + list(T.find_ntt_primes(spec.q_bits, spec.nq - 1, two_n, q0))
    else:
        qs = list(T.find_ntt_primes(spec.q_bits, spec.nq, two_n))
    sp = list(T.find_ntt_primes(spec.sp_bits, spec.K, two_n, qs)) if spec.K else []
    return qs, sp


def make_context(T, spec: Spec, rotations=(), relin=True):
    """Ring, keys and evaluator; key streams mirror the reference tests'
    fixture (keygen from Rng(seed), eval keys from rng.split(77))."""
    qs, sp = _primes(T, spec)
    ring = T.RingParams(spec.N, qs + sp, spec.K)
    ctx = T.KeyContext(ring, T.NoiseParams(3.2, spec.h), T.GadgetVector(spec.group, 0))
    ev = T.Evaluator(ctx)
    rng = T.Rng(spec.seed)
    sk, pk = ctx.keygen(rng)
    krng = rng.split(77)
    keys = T.EvalKeys()
    if relin:
        keys.relin = ctx.relin_key_gen(sk, krng)
    for k in rotations:
        g = T.rotation_exponent(ring, k)
        if not keys.has(g):
            keys.add_galois(g, ctx.galois_key_gen(sk, g, krng))
    return SimpleNamespace(T=T, spec=spec, ring=ring, ctx=ctx, ev=ev, sk=sk, pk=pk, keys=keys, primes=qs, sp=sp)


def inner_sum_rotations(slots: int):
    return [1 << i for i in range(int(math.log2(slots)))]


# ---------------------------------------------------------------------------
# Synthetic records
# ---------------------------------------------------------------------------

def linear_scores(spec: Spec, seed_offset: int = 0):
    """Linear scores s = sum_j w_j a_j, a_j ~ U{0..255} (8 attributes),
    w_j ~ U[-1,1], min-max normalised over the score's attainable range
    [sum min(w_j,0)*255, sum max(w_j,0)*255] into [0,1]; plus the threshold
    t ~ U[0.3,0.7] on that normalised scale."""
    g = np.random.Generator(np.random.PCG64(spec.seed + seed_offset))
    attrs = g.integers(0, 256, size=(spec.records, 8)).astype(np.float64)
    w = g.uniform(-1.0, 1.0, size=8)
    lo, hi = 255.0 * np.minimum(w, 0).sum(), 255.0 * np.maximum(w, 0).sum()
    scores = (attrs @ w - lo) / (hi - lo)
    t = float(g.uniform(0.3, 0.7))
    return scores, t, attrs, w


def encrypt_vector(S, values, level, rng_label, encoder=None):
    T = S.T
    enc = encoder or T.Encoder(S.ring, S.spec.slots)
    m = enc.encode_slots([complex(v) for v in values], S.spec.delta, level)
    return S.ctx.encrypt(S.sk, m, S.spec.delta, T.Rng(S.spec.seed).split(rng_label), T.Domain.slots)


def encode_host(G, S, values, level):
    """Host residues of encode_slots (multi-threaded, bit-identical)."""
    enc = G.Encoder(S.ring, S.spec.slots)
    return enc.encode_slots_host([complex(v) for v in values], S.spec.delta, level)


# ---------------------------------------------------------------------------
# Config 3: private threshold count
# ---------------------------------------------------------------------------

def config3_chain(T, spec: Spec):
    return T.build_chain(T.ThresholdParams(spec.alpha, spec.beta, list(spec.degrees), spec.epsilon))


def config3_inputs(S, ct_indices=None, scores=None, t=None):
    """Encrypted score blocks (one ciphertext per 2^15 records) + encrypted
    threshold broadcast; scientist-side encryption, level = max_level."""
    spec = S.spec
    if scores is None:
        scores, t, _, _ = linear_scores(spec)
    n = spec.slots
    lvl = S.ring.max_level()
    enc = S.T.Encoder(S.ring, n)
    idx = range(spec.n_cts) if ct_indices is None else ct_indices
    cts = [encrypt_vector(S, scores[b * n:(b + 1) * n], lvl, 100 + b, enc) for b in idx]
    ct_t = encrypt_vector(S, [t] * n, lvl, 99, enc)
    return cts, ct_t, scores, t


def config3_query(S, chain, cts, ct_t, do_inner_sum=True):
    """Reference order: per-ciphertext threshold, sum mod q, one inner_sum
    (protocol.hpp:319-323)."""
    T, ev = S.T, S.ev
    acc = None
    for ct in cts:
        o = T.eval_private_threshold_plain_norm(ev, ct, ct_t, S.spec.norm, chain, S.keys)
        acc = o if acc is None else ev.add(acc, o)
    if do_inner_sum:
        acc = T.inner_sum(ev, acc, S.spec.slots, S.keys)
    return acc
