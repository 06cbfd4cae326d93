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
