"""TTRS wire formats (reference serialize.hpp): the
B200 module writes byte-identical objects and reads the reference's."""
import numpy as np
import pytest

from common import assert_ct_equal, enc_slots, make_setup


def test_chain_bytes_match_reference_cpu(G, R):
    cg = G.build_chain(G.ThresholdParams(8, 12, [15, 15, 27], 0.0))
    cr = R.build_chain(R.ThresholdParams(8, 12, [15, 15, 27], 0.0))
    bg, br = G.serialize_chain(cg), R.serialize_chain(cr)
    assert bg == br
    back = G.deserialize_chain(br)
    assert G.serialize_chain(back) == bg
    with pytest.raises(Exception, match="bad magic"):
        G.deserialize_chain(b"XXXX" + bg[4:])


@pytest.fixture(scope="module")
def pair(G, R, gpu_available):
    kw = dict(N=256, nq=5, K=2, group_size=2, seed=77, rotations=(1,))
    return make_setup(G, **kw), make_setup(R, **kw)


@pytest.mark.gpu
def test_ciphertext_bytes_and_cross_load(G, R, pair):
    g, r = pair
    vals = np.linspace(-0.5, 0.5, 128)
    cg, cr = enc_slots(g, vals, 2.0 ** 40, G.Rng(4)), enc_slots(r, vals, 2.0 ** 40, R.Rng(4))
    for x, y in ((cg, cr), (g.ev.rescale(g.ev.mul_relin(cg, cg, g.keys)), r.ev.rescale(r.ev.mul_relin(cr, cr, r.keys)))):
        bg, br = G.serialize_ciphertext(x), R.serialize_ciphertext(y)
        assert bg == br
        assert len(bg) == G.ciphertext_size(g.ring, x.level(), 2) == R.ciphertext_size(r.ring, y.level(), 2)
        assert_ct_equal(G.deserialize_ciphertext(br, g.ring), x, "reference bytes -> B200")
        assert_ct_equal(R.deserialize_ciphertext(bg, r.ring), y, "B200 bytes -> reference")
    with pytest.raises(Exception, match="mismatch"):
        other = G.RingParams(256, list(G.find_ntt_primes(45, 5, 512)), 0)
        G.deserialize_ciphertext(G.serialize_ciphertext(cg), other)


@pytest.mark.gpu
def test_switching_key_seed_compressed(G, R, pair):
    g, r = pair
    bg, br = G.serialize_switching_key(g.keys.relin), R.serialize_switching_key(r.keys.relin)
    assert bg == br
    k = G.deserialize_switching_key(br, g.ring)  # a-parts regenerated from the seed
    for p, q in zip(k.a + k.b, g.keys.relin.a + g.keys.relin.b):
        assert np.array_equal(p.to_numpy(), q.to_numpy())
    keys = G.EvalKeys()
    keys.relin = k
    vals = np.linspace(-0.5, 0.5, 128)
    c = enc_slots(g, vals, 2.0 ** 40, G.Rng(8))
    assert_ct_equal(g.ev.mul_relin(c, c, keys), g.ev.mul_relin(c, c, g.keys), "loaded key")


@pytest.mark.gpu
def test_secret_key_bytes(G, R, pair):
    g, r = pair
    bg, br = G.serialize_secret_key(g.sk), R.serialize_secret_key(r.sk)
    assert bg == br
    sk = G.deserialize_secret_key(br, g.ring)
    assert sk.id() == g.sk.id() and list(sk.coeffs()) == list(g.sk.coeffs())


def test_hostile_counts_rejected_before_allocation(G):
    """A count read from untrusted bytes must fit the bytes that follow
    before anything is allocated (a short buffer claiming 2^32-1
    key digits must not reserve 2*w*n device words). Runs without a GPU: the
    check fires before the first device allocation."""
    import struct
    N = 64
    moduli = list(G.find_ntt_primes(40, 3, 2 * N)) + list(G.find_ntt_primes(50, 1, 2 * N))
    ring = G.RingParams(N, moduli, 1)
    hdr = struct.pack("<IHHIII", 0x54545253, 1, 2, N, len(moduli), 1) + b"".join(struct.pack("<Q", q) for q in moduli)
    body = struct.pack("<IIQQQI", 2, 0, 1, 2, 3, 0xFFFFFFFF)  # gadget, ids, a_seed, digit count
    with pytest.raises(Exception, match="truncated input"):
        G.deserialize_switching_key(hdr + body, ring)
    ct_hdr = struct.pack("<IHHIII", 0x54545253, 1, 1, N, len(moduli), 1) + b"".join(struct.pack("<Q", q) for q in moduli)
    with pytest.raises(Exception, match="truncated input"):
        G.deserialize_ciphertext(ct_hdr + struct.pack("<I", 1 << 30) + b"\0" * 25, ring)
    sk_hdr = struct.pack("<IHHIII", 0x54545253, 1, 7, N, len(moduli), 1) + b"".join(struct.pack("<Q", q) for q in moduli)
    with pytest.raises(Exception, match="truncated input"):
        G.deserialize_secret_key(sk_hdr + struct.pack("<QI", 5, 1 << 31), ring)
    chain = G.serialize_chain(G.build_chain(G.ThresholdParams(8, 12, [15], 0.0)))
    bad = bytearray(chain)
    bad[24:28] = struct.pack("<I", 0xFFFFFFF0)  # the degree count (after magic, version, kind, alpha, beta, epsilon)
    with pytest.raises(Exception, match="truncated input"):
        G.deserialize_chain(bytes(bad))
