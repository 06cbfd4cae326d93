"""GPU parity: every evaluation-path op of the B200 module against the
compiled, unmodified reference (oracle/_ref) on identical seeded inputs.
Integer work => bit-exact residues, identical level/form/scale metadata.
Reference tests mirrored: test_ring.cpp:18-119,167-224; test_rlwe.cpp:131-264,
363-416; test_ckks.cpp:164-411; test_threshold.cpp:168-233."""
import math

import numpy as np
import pytest

from common import assert_ct_equal, assert_poly_equal, dec_slots, enc_slots, make_setup

pytestmark = pytest.mark.gpu


def both(G, R, **kw):
    return make_setup(G, **kw), make_setup(R, **kw)


@pytest.fixture(scope="module")
def pair64(G, R, gpu_available):
    kw = dict(N=64, nq=8, K=2, group_size=2, seed=47, rotations=(1, 2, 3, 4, 8, 16), conj=True)
    return both(G, R, **kw)


@pytest.mark.parametrize("N", [16, 64, 256, 1024, 4096, 1 << 14, 1 << 15, 1 << 16])
def test_ntt_roundtrip_and_forward(G, R, gpu_available, N):
    primes = list(R.find_ntt_primes(50, 3, 2 * N))
    sp = list(R.find_ntt_primes(60, 1, 2 * N, primes))
    rg, rr = G.RingParams(N, primes + sp, 1), R.RingParams(N, primes + sp, 1)
    for nspecial in (0, 1):
        pg = G.sample_uniform(rg, 2, nspecial, G.Rng(N + nspecial))
        pr = R.sample_uniform(rr, 2, nspecial, R.Rng(N + nspecial))
        assert_poly_equal(pg, pr, "sample")
        fg, fr = G.ntt_transform(pg, G.Form.eval), R.ntt_transform(pr, R.Form.eval)
        assert_poly_equal(fg, fr, f"ntt fwd N={N}")
        bg = G.ntt_transform(fg, G.Form.coeff)
        assert_poly_equal(bg, pr, f"ntt roundtrip N={N}")


def test_elementwise_ops(G, R, pair64):
    g, r = pair64
    for lvl, ns in ((7, 0), (3, 2)):
        a = [T.sample_uniform(S.ring, lvl, ns, T.Rng(11)) for T, S in ((G, g), (R, r))]
        b = [T.sample_uniform(S.ring, lvl, ns, T.Rng(12)) for T, S in ((G, g), (R, r))]
        outs = []
        for (x, y) in zip(a, b):
            s = x.copy(); s.add_inplace(y)
            d = x.copy(); d.sub_inplace(y)
            n = x.copy(); n.negate_inplace()
            xe, ye = x.copy(), y.copy(); xe.ntt_forward(); ye.ntt_forward()
            m = xe.copy(); m.mul_pointwise_inplace(ye)
            acc = m.copy(); acc.mul_acc_pointwise(xe, ye)
            sc = x.copy(); sc.mul_scalar_inplace([(1 << 61) + 12345 * i for i in range(10)])
            outs.append((s, d, n, m, acc, sc))
        for name, pg, pr in zip(("add", "sub", "neg", "mul", "mac", "scalar"), outs[0], outs[1]):
            assert_poly_equal(pg, pr, name)


def test_automorphism_both_forms(G, R, pair64):
    g, r = pair64
    for form in ("coeff", "eval"):
        for gexp in (5, 25, 127, 2 * 64 - 1):
            pg = G.sample_uniform(g.ring, 7, 0, G.Rng(gexp))
            pr = R.sample_uniform(r.ring, 7, 0, R.Rng(gexp))
            if form == "eval":
                pg.ntt_forward(); pr.ntt_forward()
            assert_poly_equal(G.automorphism_apply(pg, gexp), R.automorphism_apply(pr, gexp), f"auto {form} {gexp}")


def test_rescale_round(G, R, pair64):
    g, r = pair64
    for lvl in (1, 4, 7):
        pg = G.sample_uniform(g.ring, lvl, 0, G.Rng(100 + lvl))
        pr = R.sample_uniform(r.ring, lvl, 0, R.Rng(100 + lvl))
        assert_poly_equal(G.rescale_round(pg), R.rescale_round(pr), f"rescale lvl={lvl}")


def test_keys_identical(G, R, pair64):
    g, r = pair64
    assert g.sk.id() == r.sk.id()
    assert list(g.sk.coeffs()) == list(r.sk.coeffs())
    assert_poly_equal(g.pk.b, r.pk.b, "pk.b")
    assert_poly_equal(g.pk.a, r.pk.a, "pk.a")
    for i in range(len(r.keys.relin.b)):
        assert_poly_equal(g.keys.relin.b[i], r.keys.relin.b[i], f"rlk.b[{i}]")
        assert_poly_equal(g.keys.relin.a[i], r.keys.relin.a[i], f"rlk.a[{i}]")
    for gexp in r.keys.galois_exponents():
        kg, kr = g.keys.galois_key(gexp), r.keys.galois_key(gexp)
        assert kg.a_seed == kr.a_seed and kg.from_id == kr.from_id
        assert_poly_equal(kg.b[0], kr.b[0], f"gk[{gexp}].b0")


def test_encrypt_decrypt(G, R, pair64):
    g, r = pair64
    vals = [0.1 * i - 1.5 for i in range(32)]
    cg = enc_slots(g, vals, 2.0 ** 40, G.Rng(3))
    cr = enc_slots(r, vals, 2.0 ** 40, R.Rng(3))
    assert_ct_equal(cg, cr, "encrypt")
    assert_poly_equal(g.ctx.decrypt(g.sk, cg), r.ctx.decrypt(r.sk, cr), "decrypt")
    m_g = G.Encoder(g.ring, 32).encode_slots([complex(v) for v in vals], 2.0 ** 40, 5)
    m_r = R.Encoder(r.ring, 32).encode_slots([complex(v) for v in vals], 2.0 ** 40, 5)
    assert_ct_equal(g.ctx.encrypt_pk(g.pk, m_g, 2.0 ** 40, G.Rng(4)), r.ctx.encrypt_pk(r.pk, m_r, 2.0 ** 40, R.Rng(4)),
                    "encrypt_pk")


def test_keyswitch_pieces(G, R, pair64):
    g, r = pair64
    for lvl in (7, 4, 0):
        dg = G.sample_uniform(g.ring, lvl, 0, G.Rng(200 + lvl))
        dr = R.sample_uniform(r.ring, lvl, 0, R.Rng(200 + lvl))
        digs_g, digs_r = g.ctx.decompose(dg), r.ctx.decompose(dr)
        assert len(digs_g) == len(digs_r)
        for i, (x, y) in enumerate(zip(digs_g, digs_r)):
            assert_poly_equal(x, y, f"modup lvl={lvl} digit {i}")
        xg = G.sample_uniform(g.ring, lvl, 2, G.Rng(300 + lvl))
        xr = R.sample_uniform(r.ring, lvl, 2, R.Rng(300 + lvl))
        assert_poly_equal(g.ctx.mod_down_p(xg), r.ctx.mod_down_p(xr), f"moddown lvl={lvl}")
        k0g, k1g = g.ctx.ks_inner(digs_g, g.keys.relin)
        k0r, k1r = r.ctx.ks_inner(digs_r, r.keys.relin)
        assert_poly_equal(k0g, k0r, "ks_inner c0")
        assert_poly_equal(k1g, k1r, "ks_inner c1")
        s0g, s1g = g.ctx.switch_key_apply(dg, g.keys.relin)
        s0r, s1r = r.ctx.switch_key_apply(dr, r.keys.relin)
        assert_poly_equal(s0g, s0r, "switch_key_apply c0")
        assert_poly_equal(s1g, s1r, "switch_key_apply c1")


@pytest.mark.parametrize("N,nq,K,gs", [(1024, 9, 4, 3), (1024, 22, 7, 7), (256, 20, 16, 16), (4096, 29, 10, 10),
                                        (128, 12, 5, 4)])
def test_keyswitch_pieces_tensor_core(G, R, gpu_available, monkeypatch, N, nq, K, gs):
    """ModUp / ModDown / switch_key_apply on all-FP64 rings (50-bit q and
    specials, N a multiple of 128): the int8 tensor-core base conversion
    (tg_baseconv_tc.cuh, forced on for every launch: TG_TC_BASECONV=2 is read
    when the gadget is built) vs the reference, at every digit shape (full and
    partial groups, 1..16 sources, 4..16 specials)."""
    monkeypatch.setenv("TG_TC_BASECONV", "2")
    g, r = both(G, R, N=N, nq=nq, K=K, group_size=gs, seed=91, q_bits=50, sp_bits=50)
    for lvl in sorted({nq - 1, nq // 2, 1, 0}, reverse=True):
        dg = G.sample_uniform(g.ring, lvl, 0, G.Rng(500 + lvl))
        dr = R.sample_uniform(r.ring, lvl, 0, R.Rng(500 + lvl))
        for i, (x, y) in enumerate(zip(g.ctx.decompose(dg), r.ctx.decompose(dr))):
            assert_poly_equal(x, y, f"modup N={N} lvl={lvl} digit {i}")
        xg = G.sample_uniform(g.ring, lvl, K, G.Rng(600 + lvl))
        xr = R.sample_uniform(r.ring, lvl, K, R.Rng(600 + lvl))
        assert_poly_equal(g.ctx.mod_down_p(xg), r.ctx.mod_down_p(xr), f"moddown N={N} lvl={lvl}")
        s0g, s1g = g.ctx.switch_key_apply(dg, g.keys.relin)
        s0r, s1r = r.ctx.switch_key_apply(dr, r.keys.relin)
        assert_poly_equal(s0g, s0r, f"switch_key_apply c0 N={N} lvl={lvl}")
        assert_poly_equal(s1g, s1r, f"switch_key_apply c1 N={N} lvl={lvl}")


def _pair_cts(g, r, n, delta=2.0 ** 45, seed=5, level=None):
    vals = [math.sin(0.37 * i) for i in range(n)]
    return (enc_slots(g, vals, delta, g.T.Rng(seed), level=level), enc_slots(r, vals, delta, r.T.Rng(seed), level=level),
            vals)


def test_evaluator_ops(G, R, pair64):
    g, r = pair64
    xg, xr, _ = _pair_cts(g, r, 32, seed=5)
    yg, yr, _ = _pair_cts(g, r, 32, seed=6, level=5)
    for name, fn in [
        ("add", lambda S, x, y: S.ev.add(x, y)),
        ("sub", lambda S, x, y: S.ev.sub(x, y)),
        ("mul", lambda S, x, y: S.ev.mul(x, y)),
        ("mul_relin", lambda S, x, y: S.ev.mul_relin(x, y, S.keys)),
        ("relin+rescale", lambda S, x, y: S.ev.rescale(S.ev.mul_relin(x, y, S.keys))),
        ("mul_scalar", lambda S, x, y: S.ev.mul_scalar(x, -0.318, 2.0 ** 45)),
        ("add_scalar", lambda S, x, y: S.ev.add_scalar(x, 0.75)),
        ("add_scalar_eval", lambda S, x, y: S.ev.add_scalar(S.ev.mul(x, y), -1.0)),
        ("rescale", lambda S, x, y: S.ev.rescale(x)),
        ("rotate1", lambda S, x, y: S.ev.rotate(x, 1, S.keys)),
        ("rotate3", lambda S, x, y: S.ev.rotate(y, 3, S.keys)),
        ("conjugate", lambda S, x, y: S.ev.conjugate(x, S.keys)),
    ]:
        assert_ct_equal(fn(g, xg, yg), fn(r, xr, yr), name)


def test_inplace_write_after_memoised_transform(G, R, pair64):
    """mul(a, b) memoises a's eval form on its block; a later in-place
    add/sub/negate must not reuse it (stale eval-form cache)."""
    g, r = pair64
    xg, xr, _ = _pair_cts(g, r, 32, seed=21)
    yg, yr, _ = _pair_cts(g, r, 32, seed=22)
    zg, zr, _ = _pair_cts(g, r, 32, seed=23)
    outs = []
    for S, x, y, z in ((g, xg, yg, zg), (r, xr, yr, zr)):
        a = x.copy()
        hold = a.copy()              # a shared block: mul memoises its eval form
        m1 = S.ev.mul(a, y)
        del hold                     # a's block is exclusively owned again
        a.add_inplace(z)             # in place on the block whose eval form was memoised
        m2 = S.ev.mul(a, y)
        a.sub_inplace(y)
        m3 = S.ev.mul_relin(a, z, S.keys)
        outs.append((m1, m2, m3))
    for name, cg_, cr_ in zip(("mul", "mul after add_inplace", "mul_relin after sub_inplace"), outs[0], outs[1]):
        assert_ct_equal(cg_, cr_, name)


def test_mul_plain(G, R, pair64):
    g, r = pair64
    xg, xr, _ = _pair_cts(g, r, 32, seed=8)
    vals = [0.5 + 0.01 * i for i in range(32)]
    outs = []
    for S in (g, r):
        p = S.T.Encoder(S.ring, 32).encode_slots([complex(v) for v in vals], float(S.ring.modulus(7)), 7)
        p.ntt_forward()
        outs.append(S.ev.rescale(S.ev.mul_plain(xg if S is g else xr, p, float(S.ring.modulus(7)))))
    assert_ct_equal(outs[0], outs[1], "mul_plain")


def test_chebyshev_inner_sum(G, R, pair64):
    g, r = pair64
    coeffs_rng = R.Rng(59)
    coeffs = [float(int(coeffs_rng.uniform(2001)) - 1000) / 4000.0 for _ in range(16)]
    vals = [-1.0 + i / 32.0 + 1.0 / 64.0 for i in range(32)]
    cg = enc_slots(g, vals, 2.0 ** 45, G.Rng(53))
    cr = enc_slots(r, vals, 2.0 ** 45, R.Rng(53))
    og = G.eval_chebyshev(g.ev, cg, coeffs, g.keys)
    orr = R.eval_chebyshev(r.ev, cr, coeffs, r.keys)
    assert_ct_equal(og, orr, "eval_chebyshev deg 15")
    got = dec_slots(g, og, 32).real
    for x, y in zip(vals, got):  # Clenshaw check (test_ckks.cpp:358-377)
        b1 = b2 = 0.0
        for k in range(15, 0, -1):
            b1, b2 = 2 * x * b1 - b2 + coeffs[k], b1
        assert abs(y - (x * b1 - b2 + coeffs[0])) < 2.0 ** -20
    assert_ct_equal(G.eval_chebyshev(g.ev, cg, [0.75], g.keys), R.eval_chebyshev(r.ev, cr, [0.75], r.keys), "deg0")
    assert_ct_equal(G.inner_sum(g.ev, cg, 32, g.keys), R.inner_sum(r.ev, cr, 32, r.keys), "inner_sum")


def test_private_threshold(G, R, gpu_available):
    """test_threshold.cpp:168-193 at the reference's fixture shape."""
    chain_g = G.build_chain(G.ThresholdParams(8, 12, [15, 15, 15], 1.0))
    chain_r = R.build_chain(R.ThresholdParams(8, 12, [15, 15, 15], 1.0))
    levels = chain_r.levels_required() + 1
    g, r = both(G, R, N=64, nq=levels + 1, K=2, group_size=2, seed=303)
    delta = 2.0 ** 45
    t_g = enc_slots(g, [80.0] * 16, delta, G.Rng(31), nslots=16)
    t_r = enc_slots(r, [80.0] * 16, delta, R.Rng(31), nslots=16)
    n_g = enc_slots(g, [1.0 / 144.0] * 16, delta, G.Rng(32), nslots=16)
    n_r = enc_slots(r, [1.0 / 144.0] * 16, delta, R.Rng(32), nslots=16)
    scores = [float(min(64 + i, 144)) for i in range(16)]
    s_g = enc_slots(g, scores, delta, G.Rng(33), nslots=16)
    s_r = enc_slots(r, scores, delta, R.Rng(33), nslots=16)
    og = G.eval_private_threshold(g.ev, s_g, t_g, n_g, chain_g, g.keys)
    orr = R.eval_private_threshold(r.ev, s_r, t_r, n_r, chain_r, r.keys)
    assert_ct_equal(og, orr, "eval_private_threshold")
    bits = (dec_slots(g, og, 16).real >= 0.5).astype(int)
    assert list(bits) == [int(s >= 80.0) for s in scores]
    pg = G.eval_private_threshold_plain_norm(g.ev, s_g, t_g, 1.0 / 144.0, chain_g, g.keys)
    pr = R.eval_private_threshold_plain_norm(r.ev, s_r, t_r, 1.0 / 144.0, chain_r, r.keys)
    assert_ct_equal(pg, pr, "eval_private_threshold_plain_norm")
    with pytest.raises(RuntimeError, match="insufficient levels"):
        low = enc_slots(g, [1.0] * 16, delta, G.Rng(1), nslots=16, level=4)
        G.eval_private_threshold(g.ev, low, t_g, n_g, chain_g, g.keys)


def test_error_contracts(G, pair64):
    g, _ = pair64
    c = enc_slots(g, [0.5] * 32, 2.0 ** 40, G.Rng(9), level=0)
    with pytest.raises(RuntimeError, match="exhausted"):
        g.ev.mul(c, c)
    with pytest.raises(RuntimeError, match="missing rotation key"):
        g.ev.rotate(c, 5, g.keys)
    with pytest.raises(RuntimeError, match="cannot rescale at level 0"):
        g.ev.rescale(c)


@pytest.mark.parametrize("N,nq,K,gs,bits,spbits", [(1 << 14, 8, 2, 2, 50, 60), (1 << 12, 6, 3, 3, 50, 60)])
def test_config1_shape_ops(G, R, gpu_available, N, nq, K, gs, bits, spbits):
    """Config-1 shape: 50-bit q-chain, 60-bit specials, uniform residues."""
    g, r = both(G, R, N=N, nq=nq, K=K, group_size=gs, seed=7, q_bits=bits, sp_bits=spbits, h=192, rotations=(1,))
    cts = []
    for S in (g, r):
        T = S.T
        rng = T.Rng(1234)
        out = []
        for i in range(2):
            c = T.Ciphertext()
            c.parts = [T.sample_uniform(S.ring, S.ring.max_level(), 0, rng.split(10 * i + j)) for j in range(2)]
            c.scale = 2.0 ** 50
            c.domain = T.Domain.slots
            c.sk_id = S.sk.id()
            out.append(c)
        cts.append(out)
    (a_g, b_g), (a_r, b_r) = cts
    assert_ct_equal(g.ev.mul_relin(a_g, b_g, g.keys), r.ev.mul_relin(a_r, b_r, r.keys), "tensor+relin")
    assert_ct_equal(g.ev.rescale(a_g), r.ev.rescale(a_r), "rescale")
    assert_ct_equal(g.ev.rotate(a_g, 1, g.keys), r.ev.rotate(a_r, 1, r.keys), "rotate 1")


def _is_prime(n):
    if n < 2:
        return False
    for p in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d, s = d // 2, s + 1
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):  # deterministic below 3.3e24
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


@pytest.mark.parametrize("N", [1 << 14, 1 << 15, 1 << 16])
def test_ntt_fp64_extreme_inputs(G, R, gpu_available, N):
    """The FP64 path at its bounds (q < 1.2 * 2^50): the 50-bit NTT primes
    nearest 2^50 (one each side) and the largest NTT primes below the bound,
    with inputs that maximise butterfly growth (all q-1, alternating 0/q-1,
    impulses, a ramp), forward and inverse, vs the reference NTT."""
    bound = 1351079888211148
    near = list(R.find_ntt_primes(50, 2, 2 * N))
    top, c = [], bound - bound % (2 * N) + 1
    while len(top) < 2:  # the largest NTT primes below the FP64 bound
        if c < bound and _is_prime(c):
            top.append(c)
        c -= 2 * N
    primes = near + top
    rg, rr = G.RingParams(N, primes, 0), R.RingParams(N, primes, 0)
    pats = []
    for name in ("max", "alt", "impulse", "ramp"):
        a = np.zeros((len(primes), N), dtype=np.uint64)
        for r, q in enumerate(primes):
            if name == "max":
                a[r] = q - 1
            elif name == "alt":
                a[r, ::2] = q - 1
            elif name == "impulse":
                a[r, 0] = q - 1
                a[r, N // 2] = q - 1
            else:
                a[r] = (np.arange(N, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15 % q)) % np.uint64(q)
        pats.append((name, a))
    for name, a in pats:
        lv = len(primes) - 1
        pg = G.Poly.from_numpy(rg, a, lv, G.Form.coeff)
        pr = R.Poly.from_numpy(rr, a, lv, R.Form.coeff)
        fg, fr = G.ntt_transform(pg, G.Form.eval), R.ntt_transform(pr, R.Form.eval)
        assert_poly_equal(fg, fr, f"fwd {name}")
        eg = G.Poly.from_numpy(rg, a, lv, G.Form.eval)
        er = R.Poly.from_numpy(rr, a, lv, R.Form.eval)
        assert_poly_equal(G.ntt_transform(eg, G.Form.coeff), R.ntt_transform(er, R.Form.coeff), f"inv {name}")


@pytest.mark.parametrize("N", [1024])
def test_fp64_elementwise_extreme_inputs(G, R, gpu_available, N):
    """FP64 products and the FP64 rescale at their bounds: primes nearest 2^50
    and the largest NTT primes below 1.2 * 2^50 (in both orders, so the
    dropped modulus is larger and smaller than the kept ones), residues 0,
    1, q-1, floor(q/2) and floor(q/2)+1 (the centring boundary of
    rescale_round), vs the reference."""
    bound = 1351079888211148
    near = list(R.find_ntt_primes(50, 2, 2 * N))
    top, c = [], bound - bound % (2 * N) + 1
    while len(top) < 2:
        if c < bound and _is_prime(c):
            top.append(c)
        c -= 2 * N
    for primes in (near + top, top + near, [top[0], near[0], top[1], near[1]]):
        rg, rr = G.RingParams(N, primes, 0), R.RingParams(N, primes, 0)
        lv = len(primes) - 1
        specials = lambda q: np.array([0, 1, q - 1, q // 2, q // 2 + 1, q - 2, 2, q // 2 - 1], dtype=np.uint64)
        a = np.zeros((len(primes), N), dtype=np.uint64)
        b = np.zeros((len(primes), N), dtype=np.uint64)
        g = np.random.Generator(np.random.PCG64(N + len(primes)))
        for r, q in enumerate(primes):
            sp = specials(q)
            a[r] = np.resize(sp, N)
            b[r] = np.resize(np.roll(sp, r + 1), N)
            a[r, 512:] = g.integers(0, q, N - 512, dtype=np.uint64)
        # last row sweeps the centring boundary against every other row's pattern
        ql = primes[-1]
        a[-1, :8 * 8] = np.repeat(specials(ql), 8)
        pg, pr = G.Poly.from_numpy(rg, a, lv, G.Form.eval), R.Poly.from_numpy(rr, a, lv, R.Form.eval)
        qg, qr = G.Poly.from_numpy(rg, b, lv, G.Form.eval), R.Poly.from_numpy(rr, b, lv, R.Form.eval)
        pg.mul_pointwise_inplace(qg)
        pr.mul_pointwise_inplace(qr)
        assert_poly_equal(pg, pr, "mul_pointwise extremes")
        pg, pr = G.Poly.from_numpy(rg, a, lv, G.Form.coeff), R.Poly.from_numpy(rr, a, lv, R.Form.coeff)
        assert_poly_equal(G.rescale_round(pg), R.rescale_round(pr), "rescale_round extremes")
