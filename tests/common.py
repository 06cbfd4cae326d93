"""Shared parity scaffolding. The product module (paper_2412_13269_b200.tetris)
and the compiled reference (oracle/_ref/tetris_ref) expose the same Python API,
so every scenario below is written once and run against both."""
from __future__ import annotations

import importlib
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
REF_DIR = ROOT / "oracle" / "_ref"


def load_ref():
    """Import the compiled reference oracle if it was built; else None."""
    if not any(REF_DIR.glob("tetris_ref*.so")):
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    return importlib.import_module("tetris_ref")


def chain_primes(T, N, q_bits, nq, sp_bits, K, q0_bits=None):
    """q-chain of nq primes (optionally a larger q0) plus K special primes."""
    two_n = 2 * N
    if q0_bits:
        q0 = list(T.find_ntt_primes(q0_bits, 1, two_n))
        qs = list(T.find_ntt_primes(q_bits, nq - 1, two_n, q0))
        primes = q0 + qs
    else:
        primes = list(T.find_ntt_primes(q_bits, nq, two_n))
    sp = list(T.find_ntt_primes(sp_bits, K, two_n, primes)) if K else []
    return primes, sp


def make_setup(T, N, nq, K, group_size, seed, q_bits=45, sp_bits=None, q0_bits=None, h=None,
               rotations=(), conj=False, relin=True):
    """Mirrors the reference tests' Fixture (test_ckks.cpp:12-37)."""
    primes, sp = chain_primes(T, N, q_bits, nq, sp_bits or q_bits, K, q0_bits)
    ring = T.RingParams(N, primes + sp, K)
    ctx = T.KeyContext(ring, T.NoiseParams(3.2, h if h is not None else N // 2), T.GadgetVector(group_size, 0))
    ev = T.Evaluator(ctx)
    rng = T.Rng(seed)
    sk, pk = ctx.keygen(rng)
    krng = rng.split(77)
    keys = T.EvalKeys()
    if relin:
        keys.relin = ctx.relin_key_gen(sk, krng)
    for k in rotations:
        g = T.rotation_exponent(ring, k)
        if not keys.has(g):
            keys.add_galois(g, ctx.galois_key_gen(sk, g, krng))
    if conj:
        g = T.conjugation_exponent(ring)
        keys.add_galois(g, ctx.galois_key_gen(sk, g, krng))
    return SimpleNamespace(T=T, ring=ring, ctx=ctx, ev=ev, sk=sk, pk=pk, keys=keys, rng=rng, primes=primes, sp=sp)


def ct_np(ct):
    return [p.to_numpy() for p in ct.parts]


def assert_ct_equal(a, b, what=""):
    """Bit-exact ciphertext equality: residues, level, form, scale, domain."""
    assert a.level() == b.level(), f"{what}: level {a.level()} != {b.level()}"
    assert int(a.form()) == int(b.form()), f"{what}: form mismatch"
    assert int(a.domain) == int(b.domain), f"{what}: domain mismatch"
    assert a.scale == b.scale, f"{what}: scale {a.scale!r} != {b.scale!r}"
    assert len(a.parts) == len(b.parts), f"{what}: degree mismatch"
    for i, (x, y) in enumerate(zip(ct_np(a), ct_np(b))):
        if not np.array_equal(x, y):
            bad = int((x != y).sum())
            raise AssertionError(f"{what}: part {i} differs in {bad}/{x.size} residues")


def assert_poly_equal(a, b, what=""):
    assert a.level() == b.level() and a.nspecial() == b.nspecial(), f"{what}: shape"
    assert int(a.form()) == int(b.form()), f"{what}: form"
    x, y = a.to_numpy(), b.to_numpy()
    if not np.array_equal(x, y):
        raise AssertionError(f"{what}: {int((x != y).sum())}/{x.size} residues differ")


def enc_slots(S, values, delta, rng, level=None, nslots=None):
    T = S.T
    n = nslots or len(values)
    enc = T.Encoder(S.ring, n)
    lvl = S.ring.max_level() if level is None else level
    m = enc.encode_slots([complex(v) for v in values], delta, lvl)
    return S.ctx.encrypt(S.sk, m, delta, rng, T.Domain.slots)


def dec_slots(S, ct, nslots):
    enc = S.T.Encoder(S.ring, nslots)
    return np.array(enc.decode_slots(S.ctx.decrypt(S.sk, ct), ct.scale))


def mirror_encoder(S_gpu, R):
    """S.encode for the reference side of a parity run: slot vectors are
    encoded once on the device (bit-identical to the reference Encoder,
    tests/test_gpu_encoder.py) and the residues handed to the reference, which
    skips its O(n^2) host DFT. Everything downstream runs in the reference."""
    def encode(SR, arr, scale, level):
        polys = S_gpu.encode(S_gpu, arr, scale, level)
        return [R.Poly.from_numpy(SR.ring, p.to_numpy(), level, R.Form.coeff, 0) for p in polys]
    return encode


def copy_chain(T, chain):
    """The same MinimaxChain in module T (build_chain is bit-exact across the
    two modules, test_host_cpu::test_remez_chain_bit_exact; degree-63 chains
    take ~20 s to build, so parity runs build them once)."""
    c = T.MinimaxChain()
    c.params = T.ThresholdParams(chain.params.alpha, chain.params.beta, list(chain.params.degrees),
                                 chain.params.epsilon)
    stages = []
    for s in chain.stages:
        t = T.ChainStage()
        t.degree, t.gamma, t.upper, t.cheb, t.error = s.degree, s.gamma, s.upper, list(s.cheb), s.error
        stages.append(t)
    c.stages = stages
    c.sign_error, c.achieved_beta = chain.sign_error, chain.achieved_beta
    return c
