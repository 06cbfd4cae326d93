"""explore_from_repacked (the orchestration of Alg. 2
lines 8-16, reference protocol.hpp:241-328) on the device vs the compiled
reference's own explore_from_repacked over a real ProtocolContext
(profile.hpp: the toy-small profile at N_big = 256, N_small = 64, shorter
threshold chains so the suite stays fast). The scientist's keys, query and
the repacked ciphertexts come from the reference (scientist_setup,
score_and_repack) and cross to the device through the TTRS wire format
(byte-identical readers), so both sides evaluate the same bytes. Output:
the encrypted decision bit, residue for residue."""
import pytest

from common import assert_ct_equal, copy_chain

pytestmark = pytest.mark.gpu


def _reference_run(R, rows):
    prof = R.Profile.toy_small()
    prof.th_local = R.ThresholdParams(8, 12, [7, 7], 1.0)
    prof.th_global = R.ThresholdParams(8, 12, [7], 1.0)
    pc = R.ProtocolContext(prof)
    specs = []
    n_small = pc.ring_small().degree()
    for j in range(2):
        f = R.FunctionSpec()
        f.lo, f.hi, f.out_min, f.out_max = 0.0, 8.0, 0.0, 2.0
        f.table = [float((i * (j + 1)) % 3) for i in range(n_small)]
        specs.append(f)
    setup = R.scientist_setup(pc, specs, 2.0, 3.0, 1234)
    db = R.Database()
    db.attribute_names = ["a", "b"]
    db.rows = [[float(i % 8), float((3 * i) % 8)] for i in range(rows)]
    rep = R.score_and_repack(pc, db, R.SelectionMatrix.identity(2), setup.query, setup.keys)
    out = R.explore_from_repacked(pc, rep, rows, setup.query, setup.keys)
    return prof, pc, setup, rep, out


def _device_args(G, R, prof, pc, setup, rep, rows):
    """The device side of the same call: rings and contexts from the
    reference context's moduli and profile, everything else through TTRS."""
    rs, rb = pc.ring_small(), pc.ring_big()
    ring_small = G.RingParams(rs.degree(), list(rs.moduli()), rs.special_count())
    ring_big = G.RingParams(rb.degree(), list(rb.moduli()), rb.special_count())
    ctx_big = G.KeyContext(ring_big, G.NoiseParams(3.2, prof.hw_big), G.GadgetVector(prof.gadget_group, 0))
    em = prof.evalmod
    bp = G.BootstrapParams()
    bp.slots, bp.secret_hw, bp.sparse_log_gap = rb.degree() // 2, prof.hw_big, 0
    bp.evalmod = G.EvalModConfig(em.cheb_degree, em.double_angles, em.lattice_bound, em.arcsine_degree,
                                 em.arcsine_window)
    bp.delta_input, bp.delta_evalmod = prof.delta_tv, prof.delta_evalmod
    ct_big = lambda c: G.deserialize_ciphertext(R.serialize_ciphertext(c), ring_big)  # noqa: E731
    key_big = lambda k: G.deserialize_switching_key(R.serialize_switching_key(k), ring_big)  # noqa: E731
    keys = G.EvalKeys()
    keys.relin = key_big(setup.keys.big.relin)
    for g in setup.keys.big.galois_exponents():
        keys.add_galois(g, key_big(setup.keys.big.galois_key(g)))
    q = setup.query
    keep = (ring_small, ring_big)  # rings outlive everything built on them
    return keep, [ctx_big, G.Evaluator(ctx_big), G.BootstrapEvaluator(ctx_big, bp), copy_chain(G, pc.chain_local()),
                  copy_chain(G, pc.chain_global()),
                  [G.deserialize_ciphertext(R.serialize_ciphertext(c), ring_small) for c in rep], rows,
                  ct_big(q.t0), ct_big(q.t1), ct_big(q.norm), q.small_sk_id, key_big(setup.keys.merge), keys]


@pytest.mark.parametrize("rows", [100, 300])  # one merge group / two groups (the batched local thresholds)
def test_explore_from_repacked_bit_exact(G, R, gpu_available, rows):
    prof, pc, setup, rep, want = _reference_run(R, rows)
    keep, args = _device_args(G, R, prof, pc, setup, rep, rows)
    got = G.explore_from_repacked(*args)
    assert_ct_equal(got, want, f"explore_from_repacked ({rows} rows)")


def test_explore_rejects_foreign_key(G, R, gpu_available):
    prof, pc, setup, rep, _ = _reference_run(R, 100)
    keep, args = _device_args(G, R, prof, pc, setup, rep, 100)
    args[10] = args[10] ^ 1  # small_sk_id
    with pytest.raises(Exception, match="foreign key"):
        G.explore_from_repacked(*args)
