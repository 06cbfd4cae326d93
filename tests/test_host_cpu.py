"""CPU tests of the product's host side (no GPU): the C-ABI library loads and
exports every symbol include/tetris_b200.h declares; host producers (prime
search, NTT tables, eval-order map, RNG streams, samplers, encoder residues,
Remez chain) match the reference's golden vectors bit for bit; device calls
fail loudly without a GPU (no CPU fallback)."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
G_DIR = ROOT / "tests" / "golden"


def header_symbols():
    text = (ROOT / "include" / "tetris_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(tg_\w+)\s*\(", text, re.M)))


def test_c_abi_exports_every_declared_symbol():
    from paper_2412_13269_b200 import LIB_PATH, load_c_abi
    assert LIB_PATH.exists(), "libtetris_b200.so not built"
    lib = load_c_abi()
    syms = header_symbols()
    assert len(syms) >= 40, syms
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, f"declared but not exported: {missing}"


def test_c_abi_without_device_fails_loudly():
    from paper_2412_13269_b200 import load_c_abi
    lib = load_c_abi()
    lib.tg_device_count.restype = ctypes.c_int
    if lib.tg_device_count() > 0:
        pytest.skip("a GPU is visible")
    ctx = ctypes.c_void_p()
    mod = (ctypes.c_uint64 * 2)(1152921504606830593, 1152921504606846977)
    rc = lib.tg_context_create(ctypes.byref(ctx), 0, 16, mod, 2, 1, None, None, None, None)
    assert rc < 0
    lib.tg_last_error.restype = ctypes.c_char_p
    assert b"no CUDA device" in lib.tg_last_error()


def test_product_device_ops_raise_without_gpu(G):
    if G.device_count() > 0:
        pytest.skip("a GPU is visible")
    ring = G.RingParams(64, list(G.find_ntt_primes(45, 3, 128)), 1)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        G.sample_uniform(ring, 1, 0, G.Rng(1))


@pytest.mark.parametrize("N", [64, 1024])
def test_tables_primes_order_map_match_golden(G, N):
    z = dict(np.load(G_DIR / f"ring_N{N}.npz"))
    primes = list(G.find_ntt_primes(50, 4, 2 * N))
    sp = list(G.find_ntt_primes(60, 2, 2 * N, primes))
    assert primes + sp == [int(q) for q in z["moduli"]]
    ring = G.RingParams(N, primes + sp, 2)
    for i in range(6):
        t = ring.tables(i)
        for k in ("w", "w_shoup", "winv", "winv_shoup"):
            assert np.array_equal(np.asarray(t[k]), z[f"t{i}_{k}"]), (i, k)
        assert [t["psi"], t["n_inv"], t["n_inv_shoup"]] == [int(v) for v in z[f"t{i}_scalars"]]
    assert np.array_equal(ring.eval_exp_table(), z["eval_exp"])
    assert np.array_equal(ring.slot_of_exp_table(), z["slot_of_exp"])
    # sampler streams: same draws as the reference's samplers
    assert np.array_equal(G.sample_uniform_host(ring, 3, 2, G.Rng(11)), z["x"])
    g = np.array(G.sample_gaussian_coeffs(N, 3.2, G.Rng(13)), dtype=np.int64)
    assert np.array_equal(g % np.int64(primes[0]), z["gauss"][0].astype(np.int64))
    t = np.array(G.sample_ternary_coeffs(N, N // 4, G.Rng(14)), dtype=np.int64)
    assert np.array_equal(t % np.int64(primes[0]), z["ternary"][0].astype(np.int64))


def test_rng_streams_match_reference(G, R):
    a, b = G.Rng(0x1234), R.Rng(0x1234)
    assert [a.next() for _ in range(50)] == [b.next() for _ in range(50)]
    a, b = a.split(9), b.split(9)
    assert [a.uniform(997) for _ in range(200)] == [b.uniform(997) for _ in range(200)]
    assert [a.normal() for _ in range(101)] == [b.normal() for _ in range(101)]


@pytest.mark.parametrize("degrees,alpha", [([15, 15, 15], 8), ([15, 15, 27], 8), ([7, 15], 6)])
def test_remez_chain_bit_exact(G, R, degrees, alpha):
    cg = G.build_chain(G.ThresholdParams(alpha, 12, degrees, 0.0))
    cr = R.build_chain(R.ThresholdParams(alpha, 12, degrees, 0.0))
    assert cg.levels_required() == cr.levels_required()
    assert cg.achieved_beta == cr.achieved_beta and cg.sign_error == cr.sign_error
    for i, (a, b) in enumerate(zip(cg.stages, cr.stages)):
        assert list(a.cheb) == list(b.cheb) and a.error == b.error and a.upper == b.upper and a.gamma == b.gamma
        assert list(cg.eval_coeffs(i)) == list(cr.eval_coeffs(i))


def test_threshold_chain_matches_golden(G):
    z = dict(np.load(G_DIR / "threshold_N64.npz"))
    c = G.build_chain(G.ThresholdParams(8, 12, [15, 15, 15], 1.0))
    assert c.levels_required() == int(z["levels_required"][0])
    for i in range(3):
        assert np.array_equal(np.array(c.eval_coeffs(i)), z[f"stage{i}_eval_coeffs"])


def test_encoder_host_residues_match_reference(G, R):
    N = 256
    primes = list(R.find_ntt_primes(45, 3, 2 * N))
    rg, rr = G.RingParams(N, primes, 0), R.RingParams(N, primes, 0)
    vals = [complex(np.sin(i), np.cos(3 * i)) for i in range(64)]
    host = G.Encoder(rg, 64).encode_slots_host(vals, 2.0 ** 30, 2)
    ref = R.Encoder(rr, 64).encode_slots(vals, 2.0 ** 30, 2).to_numpy()
    assert np.array_equal(host, ref)


def test_workload_specs_consistent(G):
    from paper_2412_13269_b200 import workloads as W
    s3 = W.CONFIGS[3]
    chain = W.config3_chain(G, s3)
    assert chain.levels_required() == 17 and s3.nq - 1 >= 17
    assert -(-s3.nq // s3.group) == 3  # dnum
    assert s3.records == s3.n_cts * s3.slots
    scores, t, _, _ = W.linear_scores(s3)
    assert 0.0 <= scores.min() and scores.max() <= 1.0 and 0.3 <= t <= 0.7
    assert 0 < (scores >= t).sum() < s3.records
