"""Pins the CPU restatement oracle (oracle/tetris_oracle.c + restatement.py)
against golden vectors produced by the compiled, unmodified reference
(tests/golden/gen_golden.py). CPU only."""
from pathlib import Path

import numpy as np
import pytest

from oracle import restatement as O

G_DIR = Path(__file__).resolve().parent / "golden"


def load(name):
    return dict(np.load(G_DIR / name))


def gct(z, prefix):
    lvl, form, dom, nparts = (int(v) for v in z[f"{prefix}_meta"])
    scale, noise = z[f"{prefix}_scale"]
    return O.OCt([z[f"{prefix}_p{i}"].copy() for i in range(nparts)], lvl, "eval" if form else "coeff", float(scale),
                 dom, int(z[f"{prefix}_skid"][0]), float(noise))


def gkey(z, prefix):
    return O.OKey(list(z[f"{prefix}_b"]), list(z[f"{prefix}_a"]), int(z[f"{prefix}_ids"][1]))


def assert_oct(got: O.OCt, z, prefix):
    want = gct(z, prefix)
    assert got.level == want.level, prefix
    assert got.form == want.form, prefix
    assert got.scale == want.scale, f"{prefix}: scale {got.scale!r} vs {want.scale!r}"
    assert len(got.parts) == len(want.parts)
    for i, (a, b) in enumerate(zip(got.parts, want.parts)):
        assert np.array_equal(a, b), f"{prefix} part {i}: {(a != b).sum()} residues differ"


def ks_noise(N, digits_max):
    return 6.0 * 3.2 * np.sqrt(float(N)) * float(digits_max)


@pytest.mark.parametrize("N", [64, 1024])
def test_ring_tables_and_ops(N):
    z = load(f"ring_N{N}.npz")
    moduli = [int(q) for q in z["moduli"]]
    ring = O.Ring(N, moduli, int(z["K"][0]))
    for i in range(len(moduli)):
        t = ring.tab[i]
        for k in ("w", "w_shoup", "winv", "winv_shoup"):
            assert np.array_equal(t[k], z[f"t{i}_{k}"]), (i, k)
        assert [t["psi"], t["n_inv"], t["n_inv_shoup"]] == [int(v) for v in z[f"t{i}_scalars"]]
    assert np.array_equal(ring.eval_exp, z["eval_exp"])
    assert np.array_equal(ring.slot_of_exp, z["slot_of_exp"])
    assert np.array_equal(ring.ntt(z["x"], 3, 2), z["x_ntt"])
    assert np.array_equal(ring.ntt(z["x_ntt"], 3, 2, inverse=True), z["x"])
    ev = O.Evaluator(ring, 2)
    assert np.array_equal(ev.automorphism(z["x"], 5, 3), z["x_auto5"])
    assert np.array_equal(ev.automorphism(z["x"], 2 * N - 1, 3), z["x_auto_conj"])
    assert np.array_equal(ev.automorphism(z["x_ntt"], 25, 3, eval_form=True), z["x_ntt_auto25"])
    y = O.OCt([z["y"]], 3, "coeff", 1.0)
    assert np.array_equal(ev.rescale(y).parts[0], z["y_rescale"])


def test_prime_search_matches():
    z = load("ring_N1024.npz")
    primes = O.find_ntt_primes(50, 4, 2048)
    sp = O.find_ntt_primes(60, 2, 2048, primes)
    assert primes + sp == [int(q) for q in z["moduli"]]


@pytest.fixture(scope="module")
def ev64():
    z = load("eval_N64.npz")
    ring = O.Ring(64, [int(q) for q in z["moduli"]], 2)
    return z, O.Evaluator(ring, int(z["group"][0]))


def test_keyswitch_pieces(ev64):
    z, ev = ev64
    rlk = gkey(z, "rlk")
    for lvl in (7, 4, 0):
        digs = ev.decompose(z[f"d{lvl}"], lvl)
        assert np.array_equal(np.stack(digs), z[f"d{lvl}_digits"]), lvl
        k0, k1 = ev.ks_inner(digs, rlk, lvl)
        assert np.array_equal(k0, z[f"d{lvl}_ks0"]) and np.array_equal(k1, z[f"d{lvl}_ks1"]), lvl
        assert np.array_equal(ev.mod_down(z[f"md{lvl}_in"], lvl), z[f"md{lvl}_out"]), lvl


def test_evaluator_ops(ev64):
    z, ev = ev64
    rlk = gkey(z, "rlk")
    gk = {int(g): gkey(z, f"gk{int(g)}") for g in z["gexps"]}
    x, y = gct(z, "x"), gct(z, "y")
    ksn = ks_noise(64, 4)
    assert_oct(ev.mul(x, y), z, "mul")
    assert_oct(ev.mul_relin(x, y, rlk, ksn), z, "mul_relin")
    assert_oct(ev.rescale(x), z, "rescale")
    assert_oct(ev.add(x, y), z, "add")
    assert_oct(ev.sub(x, y), z, "sub")
    assert_oct(ev.mul_scalar(x, -0.318, 2.0 ** 45), z, "mul_scalar")
    assert_oct(ev.add_scalar(x, 0.75), z, "add_scalar")
    assert_oct(ev.add_scalar(ev.mul(x, y), -1.0), z, "add_scalar_eval")
    assert_oct(ev.rotate(x, 1, gk, ksn), z, "rotate1")
    assert_oct(ev.rotate(y, 3, gk, ksn), z, "rotate3")
    assert_oct(ev.apply_galois(x, 127, gk[127], ksn), z, "conjugate")
    assert_oct(O.eval_chebyshev(ev, x, list(z["cheb_coeffs"]), rlk, ksn), z, "cheb15")
    assert_oct(O.inner_sum(ev, x, 32, gk, ksn), z, "inner_sum")


def test_threshold_plain_norm():
    z = load("threshold_N64.npz")
    ring = O.Ring(64, [int(q) for q in z["moduli"]], 2)
    ev = O.Evaluator(ring, 2)
    rlk = gkey(z, "rlk")
    nd = (ring.nq - 1 + 2) // 2
    stages = [list(z[f"stage{i}_eval_coeffs"]) for i in range(3)]
    out = O.threshold_plain_norm(ev, gct(z, "s"), gct(z, "t"), 1.0 / 144.0, stages, int(z["levels_required"][0]), 1.0,
                                 rlk, ks_noise(64, nd))
    assert_oct(out, z, "out_plain_norm")


def test_round_half_away():
    for x, want in [(2.5, 3), (-2.5, -3), (0.49999999999999994, 0), (2.0 ** 53 + 2, 2 ** 53 + 2), (-2.5e15 - 0.5, -2500000000000001)]:
        assert O.round_half_away(x) == want
