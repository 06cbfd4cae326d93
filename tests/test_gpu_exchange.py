"""The device side of the multi-GPU exchange (bench.py
reduce_partial_to_root), exercised on one GPU: R per-rank partial
ciphertexts are summed as wrapping 64-bit integers exactly as NCCL's
ncclUint64/int64 SUM does, the sum is uploaded, and the product's mod-q
fix-up (ciphertext_reduce_inplace -> tg_poly_reduce) must give the
sequential mod-q sum (Evaluator::add, ckks.hpp:201-217) bit for bit; the
rank-0 inner_sum of it equals the reference's inner_sum of the reference's
sum (protocol.hpp:319-323)."""
import dataclasses

import numpy as np
import pytest

from common import assert_ct_equal
from paper_2412_13269_b200 import distributed as D
from paper_2412_13269_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pair(G, R, gpu_available):
    spec = dataclasses.replace(W.CONFIGS[4], N=1024, records=1024, n_cts=1)
    rot = W.inner_sum_rotations(spec.slots)
    return spec, W.make_context(G, spec, rotations=rot), W.make_context(R, spec, rotations=rot)


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("level", [1, 4])
def test_partial_reduce_then_inner_sum(G, R, pair, world, level):
    spec, g, r = pair
    D.check_exact(world, g.primes)
    rng = np.random.default_rng(7 * world + level)
    vecs = [rng.uniform(0.0, 1.0, spec.slots) for _ in range(world)]
    labels = [1000 + i for i in range(world)]
    pg = W.encrypt_many(g, vecs, level, labels)   # rank i's partial
    pr = W.encrypt_many(r, vecs, level, labels)
    for a, b in zip(pg, pr):
        assert_ct_equal(a, b, "partials")
    # NCCL SUM over int64 / uint64 words: wrapping 64-bit addition
    words = np.stack([np.stack([p.to_numpy() for p in c.parts]) for c in pg])
    summed = words.sum(axis=0, dtype=np.uint64)
    ct = G.ciphertext_from_numpy(g.ring, np.ascontiguousarray(summed), level, pg[0].form(), pg[0].scale,
                                 pg[0].domain, pg[0].sk_id)
    G.ciphertext_reduce_inplace(ct)
    want = pr[0]
    for c in pr[1:]:
        want = r.ev.add(want, c)
    got = np.stack([p.to_numpy() for p in ct.parts])
    assert np.array_equal(got, np.stack([p.to_numpy() for p in want.parts])), "device mod-q fix-up"
    cg = G.inner_sum(g.ev, ct, spec.slots, g.keys)
    cr = R.inner_sum(r.ev, want, spec.slots, r.keys)
    assert np.array_equal(np.stack([p.to_numpy() for p in cg.parts]), np.stack([p.to_numpy() for p in cr.parts]))
