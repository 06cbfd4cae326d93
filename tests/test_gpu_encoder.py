"""GPU slot encoder (tg_encode_slots) against the reference Encoder
(ckks.hpp:59-86, 137-142): bit-exact residues for every stride/level, batched
launches, the level-0 overflow contract, and a full config-2/4 size vector."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rings(G, R, N, nq, bits=45):
    primes = list(R.find_ntt_primes(bits, nq, 2 * N))
    return G.RingParams(N, primes, 0), R.RingParams(N, primes, 0)


def _values(n, seed, mag=1.0):
    g = np.random.Generator(np.random.PCG64(seed))
    return mag * (g.uniform(-1, 1, n) + 1j * g.uniform(-1, 1, n))


@pytest.mark.parametrize("N,n,level", [(64, 32, 2), (256, 64, 0), (256, 64, 2), (1024, 512, 3), (4096, 256, 1)])
def test_encode_matches_reference(G, R, gpu_available, N, n, level):
    rg, rr = _rings(G, R, N, 4)
    vals = list(_values(n, N + n + level, mag=3.0))
    gpu = G.Encoder(rg, n).encode_slots(vals, 2.0 ** 30, level).to_numpy()
    ref = R.Encoder(rr, n).encode_slots(vals, 2.0 ** 30, level).to_numpy()
    assert gpu.shape == ref.shape
    assert np.array_equal(gpu, ref)


def test_encode_many_matches_single(G, R, gpu_available):
    N, n = 1 << 12, 1 << 11
    rg, rr = _rings(G, R, N, 3)
    batch = np.stack([_values(n, 100 + b) for b in range(5)])  # not a multiple of the per-thread batch
    enc = G.Encoder(rg, n)
    many = enc.encode_slots_many(batch, 2.0 ** 40, 2)
    renc = R.Encoder(rr, n)
    for b in range(5):
        ref = renc.encode_slots(list(batch[b]), 2.0 ** 40, 2).to_numpy()
        assert np.array_equal(many[b].to_numpy(), ref), f"vector {b}"


def test_encode_rejects_overflow_and_bad_length(G, gpu_available):
    N = 256
    primes = list(G.find_ntt_primes(30, 2, 2 * N))
    enc = G.Encoder(G.RingParams(N, primes, 0), 64)
    with pytest.raises(Exception, match="overflows"):
        enc.encode_slots([complex(1e6, 0)] * 64, 2.0 ** 20, 0)
    with pytest.raises(Exception, match="length"):
        enc.encode_slots([0j] * 63, 2.0 ** 20, 1)


def test_encode_full_size_record_block(G, R, gpu_available):
    """One config-2 attribute column (2^14 slots at N=2^15) vs the reference,
    and the config-3/4 block size (2^15 slots at N=2^16) vs the host encoder
    (multi-threaded restatement pinned to the reference above and in
    test_host_cpu; the single-threaded reference takes ~15 s there)."""
    for N, bits in ((1 << 15, 40), (1 << 16, 50)):
        n = N // 2
        rg, rr = _rings(G, R, N, 2, bits)
        g = np.random.Generator(np.random.PCG64(N))
        vals = g.integers(0, 256, n) / (8 * 255.0) + 0j
        enc = G.Encoder(rg, n)
        enc.encode_slots(list(vals[:n]), 2.0 ** bits, 1)  # warm (table upload)
        t0 = time.perf_counter()
        gpu = enc.encode_slots(list(vals), 2.0 ** bits, 1).to_numpy()
        t_gpu = time.perf_counter() - t0
        t0 = time.perf_counter()
        if N == 1 << 15:
            ref = R.Encoder(rr, n).encode_slots(list(vals), 2.0 ** bits, 1).to_numpy()
        else:
            ref = enc.encode_slots_host(list(vals), 2.0 ** bits, 1)
        t_ref = time.perf_counter() - t0
        print(f"encode n={n}: gpu {t_gpu * 1e3:.1f} ms, reference {t_ref * 1e3:.0f} ms")
        assert np.array_equal(gpu, ref)
