"""PFE scoring, ring repacking and ring merge/split (
reference pfe.hpp, repack.hpp, rlwe.hpp:684-802) on the device vs the
compiled reference: identical ciphertexts, traces and automorphism counts."""
import numpy as np
import pytest

from common import assert_ct_equal

pytestmark = pytest.mark.gpu


def _ctx(T, N, primes, K, gs, seed, h=None):
    ring = T.RingParams(N, primes, K)
    ctx = T.KeyContext(ring, T.NoiseParams(3.2, h or N // 2), T.GadgetVector(gs, 0))
    rng = T.Rng(seed)
    sk, _ = ctx.keygen(rng)
    return ring, ctx, sk, rng


def _specs(T, N, ncols, seed):
    g = np.random.Generator(np.random.PCG64(seed))
    out = []
    for c in range(ncols):
        s = T.FunctionSpec()
        s.lo, s.hi = float(c), float(c + 10)
        s.table = list(g.uniform(-1, 1, N))
        out.append(s)
    return out


def test_pfe_eval_scores_bit_exact(G, R, gpu_available):
    N = 64
    primes = list(R.find_ntt_primes(50, 2, 2 * N))
    sides = {}
    for T in (G, R):
        ring, ctx, sk, rng = _ctx(T, N, primes, 0, 1, 5)
        tvs = [T.build_test_vector(ctx, s, sk, 2.0 ** 30, rng.split(10 + i)) for i, s in enumerate(_specs(T, N, 3, 9))]
        g = np.random.Generator(np.random.PCG64(3))
        rows = [[float(c + g.uniform(0, 10)) for c in range(3)] for _ in range(12)]
        rows[0][0] = 9.999999  # rounds up to n: clamped to n-1
        sides[T] = (T.eval_scores(rows, tvs, True), tvs, ctx, sk, ring)
    (og, tg), tvs_g, ctx_g, sk_g, ring_g = sides[G]
    (orr, tr), tvs_r, *_ = sides[R]
    assert list(tg) == list(tr)
    assert len(og) == len(orr) == 12
    for a, b in zip(og, orr):
        assert_ct_equal(a, b, "eval_scores")
    for i in (0, 2):
        for e in (0, 7, 63, 64, 100):
            assert_ct_equal(G.lookup(tvs_g[i], e), R.lookup(tvs_r[i], e), f"lookup {e}")
    with pytest.raises(Exception, match="out of domain"):
        G.eval_scores([[100.0, 1.0, 2.0]], tvs_g)
    with pytest.raises(Exception, match="attributes, expected"):
        G.eval_scores([[1.0]], tvs_g)


def test_repack_bit_exact(G, R, gpu_available):
    N = 64
    primes = list(R.find_ntt_primes(45, 3, 2 * N))
    sp = list(R.find_ntt_primes(50, 2, 2 * N, primes))
    outs = {}
    for T in (G, R):
        ring, ctx, sk, rng = _ctx(T, N, primes + sp, 2, 2, 11)
        keys = T.gen_repack_keys(ctx, sk, rng.split(3))
        cts = []
        for i in range(40):
            if i % 7 == 3:
                cts.append(None)
                continue
            m = T.poly_from_i64(ring, [i * 1000 - 20000] + [0] * (N - 1), ring.max_level())
            cts.append(ctx.encrypt(sk, m, 2.0 ** 20, rng.split(100 + i), T.Domain.coeffs))
        outs[T] = T.repack(ctx, cts, keys)
    (cg, ng), (cr, nr) = outs[G], outs[R]
    assert ng == nr
    assert_ct_equal(cg, cr, "repack")


def test_ring_merge_and_split_bit_exact(G, R, gpu_available):
    n_small, n_big = 32, 128
    primes = list(R.find_ntt_primes(45, 3, 2 * n_big))
    sp = list(R.find_ntt_primes(50, 2, 2 * n_big, primes))
    res = {}
    for T in (G, R):
        small, sctx, ssk, srng = _ctx(T, n_small, primes[:2] + sp, 2, 2, 21)
        big, bctx, bsk, brng = _ctx(T, n_big, primes + sp, 2, 2, 22)
        emb = T.embed_secret(ssk, big, n_big // n_small)
        swk = bctx.switch_key_gen(emb, bsk, brng.split(1))
        cts = []
        for i in range(4):
            m = T.poly_from_i64(small, list(range(i, i + n_small)), 1)
            cts.append(sctx.encrypt(ssk, m, 2.0 ** 20, srng.split(30 + i), T.Domain.coeffs))
        merged = T.ring_merge_many(bctx, [cts[0], None, cts[2], cts[3]], swk)
        # split: big -> half ring (stride 2)
        half, hctx, hsk, hrng = _ctx(T, n_big // 2, primes[:2] + sp, 2, 2, 23)
        emb2 = T.embed_secret(hsk, big, 2)
        to_emb = bctx.switch_key_gen(bsk, emb2, brng.split(2))
        m2 = T.poly_from_i64(big, list(range(n_big)), 1)
        ctb = bctx.encrypt(bsk, m2, 2.0 ** 20, brng.split(40), T.Domain.coeffs)
        even, odd = T.ring_split(bctx, half, ctb, to_emb, hsk.id())
        back = T.ring_merge(bctx, even, odd, bctx.switch_key_gen(emb2, bsk, brng.split(3)))
        res[T] = (merged, even, odd, back)
    for name, a, b in zip(("merge_many", "split even", "split odd", "merge back"), res[G], res[R]):
        assert_ct_equal(a, b, name)


def test_base2_gadget_keyswitch_bit_exact(G, R, gpu_available):
    """Base-2^b gadget refinement (rlwe.hpp:103-135; the small-ring profile's
    small_base2 = 30): single-prime groups split into balanced sub-digits."""
    N = 64
    primes = list(R.find_ntt_primes(55, 1, 2 * N)) + list(R.find_ntt_primes(54, 2, 2 * N, R.find_ntt_primes(55, 1, 2 * N)))
    sp = list(R.find_ntt_primes(60, 1, 2 * N, primes))
    outs = {}
    for T in (G, R):
        ring = T.RingParams(N, primes + sp, 1)
        ctx = T.KeyContext(ring, T.NoiseParams(3.2, 32), T.GadgetVector(1, 30))
        rng = T.Rng(17)
        sk, _ = ctx.keygen(rng)
        keys = T.gen_repack_keys(ctx, sk, rng.split(3))
        relin = ctx.relin_key_gen(sk, rng.split(4))
        cts = []
        for i in range(6):
            m = T.poly_from_i64(ring, [i * 100 + 7] + [0] * (N - 1), ring.max_level())
            cts.append(ctx.encrypt(sk, m, 2.0 ** 20, rng.split(100 + i), T.Domain.coeffs))
        ev = T.Evaluator(ctx)
        ek = T.EvalKeys()
        ek.relin = relin
        outs[T] = (T.repack(ctx, cts, keys)[0], ev.mul_relin(cts[1], cts[2], ek), ctx, ring)
    for name, a, b in zip(("repack", "mul_relin"), outs[G][:2], outs[R][:2]):
        assert_ct_equal(a, b, f"base2 {name}")
