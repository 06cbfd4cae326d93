"""BASELINE.json workloads (configs 1-5), written once against the shared
Python API so the same code drives the B200 module and the compiled reference
(oracle/_ref, test/bench checker only).

Synthetic data (there is no dataset): every record attribute is drawn from a
seeded numpy PCG64 stream with BASELINE.json's distributions; the reference's
own Rng drives keys, noise and encryption randomness. Parameter choices left
open by BASELINE.json are fixed here and documented in DESIGN.md.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from types import SimpleNamespace

import os

import numpy as np


@dataclass(frozen=True)
class Spec:
    name: str
    N: int
    nq: int                 # q-chain length (max_level + 1)
    q_bits: int             # arithmetic primes (~= log2 Delta)
    K: int                  # special primes
    sp_bits: int
    group: int              # gadget group size (dnum = ceil(nq / group))
    h: int                  # secret Hamming weight
    delta_log2: int
    q0_bits: int | None = None
    degrees: tuple = ()
    alpha: int = 8
    beta: int = 12
    epsilon: float = 0.0
    norm: float = 1.0
    n_cts: int = 1
    records: int = 0
    seed: int = 0x7e7215

    @property
    def slots(self) -> int:
        return self.N // 2

    @property
    def delta(self) -> float:
        return float(2 ** self.delta_log2)


CONFIGS = {
    # configs[0]: ring-op microbench, 64 ciphertexts of uniform residues
    1: Spec("config1-ringops", N=1 << 14, nq=8, q_bits=50, K=2, sp_bits=60, group=2, h=192, delta_log2=50,
            n_cts=64, records=0, seed=0xC0F1),
    # configs[1]: encrypted linear score, 2^16 records x 8 attributes
    2: Spec("config2-linear-score", N=1 << 15, nq=4, q_bits=40, q0_bits=60, K=1, sp_bits=60, group=4, h=192,
            delta_log2=40, n_cts=4, records=1 << 16, seed=0xC0F2),
    # configs[2]: private threshold count, 2^17 records, (15,15,27)
    3: Spec("config3-threshold-count", N=1 << 16, nq=21, q_bits=50, K=7, sp_bits=50, group=7, h=192,
            delta_log2=50, degrees=(15, 15, 27), alpha=8, epsilon=0.0, norm=1.0, n_cts=4, records=1 << 17,
            seed=0xC0F3),
    # configs[3]: full TETRIS statement, 2^18 records: three private thresholds
    # (blood sugar, blood pressure, 8-attribute encrypted linear risk score),
    # AND by products, plaintext disorder flag, slot-sum. Levels: the
    # thresholds take 17 from L (risk score: from L-1 after its rescale), two
    # AND products + the flag product take 3 more -> count at level L-20 = 1
    # (two limbs for decoding, ckks.hpp:121-134) with L = 21.
    4: Spec("config4-tetris-statement", N=1 << 16, nq=22, q_bits=50, K=7, sp_bits=50, group=7, h=192,
            delta_log2=50, degrees=(15, 15, 27), alpha=8, epsilon=0.0, norm=1.0, n_cts=8, records=1 << 18,
            seed=0xC0F4),
    # configs[4]: scale-out stress, 2^20 records (32 record blocks), three
    # degree-63 stages (levels_required 22), L = 28, dnum = 3 (group 10:
    # 10 x 50-bit digits under P = 10 x 50-bit specials, so every modulus
    # takes the FP64 path). Count at level 3.
    5: Spec("config5-stress", N=1 << 16, nq=29, q_bits=50, K=10, sp_bits=50, group=10, h=192,
            delta_log2=50, degrees=(63, 63, 63), alpha=13, epsilon=0.0, norm=1.0, n_cts=32, records=1 << 20,
            seed=0xC0F5),
}


def _primes(T, spec: Spec):
    two_n = 2 * spec.N
    if spec.q0_bits:
        q0 = list(T.find_ntt_primes(spec.q0_bits, 1, two_n))
        qs = q0 + list(T.find_ntt_primes(spec.q_bits, spec.nq - 1, two_n, q0))
    else:
        qs = list(T.find_ntt_primes(spec.q_bits, spec.nq, two_n))
    sp = list(T.find_ntt_primes(spec.sp_bits, spec.K, two_n, qs)) if spec.K else []
    return qs, sp


def make_context(T, spec: Spec, rotations=(), relin=True):
    """Ring, keys and evaluator; key streams mirror the reference tests'
    fixture (keygen from Rng(seed), eval keys from rng.split(77))."""
    qs, sp = _primes(T, spec)
    ring = T.RingParams(spec.N, qs + sp, spec.K)
    ctx = T.KeyContext(ring, T.NoiseParams(3.2, spec.h), T.GadgetVector(spec.group, 0))
    ev = T.Evaluator(ctx)
    rng = T.Rng(spec.seed)
    sk, pk = ctx.keygen(rng)
    krng = rng.split(77)
    keys = T.EvalKeys()
    if relin:
        keys.relin = ctx.relin_key_gen(sk, krng)
    for k in rotations:
        g = T.rotation_exponent(ring, k)
        if not keys.has(g):
            keys.add_galois(g, ctx.galois_key_gen(sk, g, krng))
    return SimpleNamespace(T=T, spec=spec, ring=ring, ctx=ctx, ev=ev, sk=sk, pk=pk, keys=keys, primes=qs, sp=sp,
                           encode=encode_slots_batch)


def encode_slots_batch(S, arr, scale, level):
    """Encoder::encode_slots of every row of `arr` ([batch][slots] complex):
    one device launch on the B200 module, the per-vector host DFT elsewhere.
    Parity harnesses may replace S.encode to feed the reference the device
    encoder's (bit-identical) residues instead of re-running its O(n^2) DFT."""
    enc = S.T.Encoder(S.ring, S.spec.slots)
    if hasattr(enc, "encode_slots_many"):
        return list(enc.encode_slots_many(arr, scale, level))
    return [enc.encode_slots(list(v), scale, level) for v in arr]


def inner_sum_rotations(slots: int):
    return [1 << i for i in range(int(math.log2(slots)))]


# ---------------------------------------------------------------------------
# Synthetic records
# ---------------------------------------------------------------------------

def linear_scores(spec: Spec, seed_offset: int = 0):
    """Linear scores s = sum_j w_j a_j, a_j ~ U{0..255} (8 attributes),
    w_j ~ U[-1,1], min-max normalised over the score's attainable range
    [sum min(w_j,0)*255, sum max(w_j,0)*255] into [0,1]; plus the threshold
    t ~ U[0.3,0.7] on that normalised scale."""
    g = np.random.Generator(np.random.PCG64(spec.seed + seed_offset))
    attrs = g.integers(0, 256, size=(spec.records, 8)).astype(np.float64)
    w = g.uniform(-1.0, 1.0, size=8)
    lo, hi = 255.0 * np.minimum(w, 0).sum(), 255.0 * np.maximum(w, 0).sum()
    scores = (attrs @ w - lo) / (hi - lo)
    t = float(g.uniform(0.3, 0.7))
    return scores, t, attrs, w


def encrypt_vector(S, values, level, rng_label, encoder=None):
    T = S.T
    enc = encoder or T.Encoder(S.ring, S.spec.slots)
    m = enc.encode_slots([complex(v) for v in values], S.spec.delta, level)
    return S.ctx.encrypt(S.sk, m, S.spec.delta, T.Rng(S.spec.seed).split(rng_label), T.Domain.slots)


def encode_host(G, S, values, level):
    """Host residues of encode_slots (multi-threaded, bit-identical)."""
    enc = G.Encoder(S.ring, S.spec.slots)
    return enc.encode_slots_host([complex(v) for v in values], S.spec.delta, level)


# ---------------------------------------------------------------------------
# Config 3: private threshold count
# ---------------------------------------------------------------------------

def config3_chain(T, spec: Spec):
    return T.build_chain(T.ThresholdParams(spec.alpha, spec.beta, list(spec.degrees), spec.epsilon))


def config3_inputs(S, ct_indices=None, scores=None, t=None):
    """Encrypted score blocks (one ciphertext per 2^15 records) + encrypted
    threshold broadcast; scientist-side encryption, level = max_level."""
    spec = S.spec
    if scores is None:
        scores, t, _, _ = linear_scores(spec)
    n = spec.slots
    lvl = S.ring.max_level()
    enc = S.T.Encoder(S.ring, n)
    idx = range(spec.n_cts) if ct_indices is None else ct_indices
    cts = [encrypt_vector(S, scores[b * n:(b + 1) * n], lvl, 100 + b, enc) for b in idx]
    ct_t = encrypt_vector(S, [t] * n, lvl, 99, enc)
    return cts, ct_t, scores, t


def config3_query(S, chain, cts, ct_t, do_inner_sum=True):
    """Reference order: per-ciphertext threshold, sum mod q, one inner_sum
    (protocol.hpp:319-323)."""
    T, ev = S.T, S.ev
    acc = None
    for ct in cts:
        o = T.eval_private_threshold_plain_norm(ev, ct, ct_t, S.spec.norm, chain, S.keys)
        acc = o if acc is None else ev.add(acc, o)
    if do_inner_sum:
        acc = T.inner_sum(ev, acc, S.spec.slots, S.keys)
    return acc


def run_concurrent(T, ring, fn, items, streams):
    """fn(item) for every item; with the B200 module and streams > 1 the items
    are spread round-robin over `streams` host threads, each issuing on its
    own CUDA stream (stream_scope). Fork and join are device-side events, not
    host synchronisations: each worker stream first waits for the caller's
    stream (the inputs it made), and the caller's stream waits for every
    worker stream before anything later runs on it, so the host keeps issuing
    while the GPU works. Results come back in item order, so every later
    reduction runs in the reference's order."""
    items = list(items)
    if streams <= 1 or len(items) <= 1:
        return [fn(x) for x in items]
    import contextlib
    import threading
    out = [None] * len(items)
    errs = []
    k = min(streams, len(items))
    scoped = hasattr(T, "stream_scope")  # the CPU reference: plain threads (protocol.hpp:297-311)
    if scoped:
        fork = T.StreamEvent(ring)
        fork.record()  # the caller's stream: inputs made so far
        done = [T.StreamEvent(ring) for _ in range(k)]

    def worker(w):
        try:
            with (T.stream_scope(ring, w) if scoped else contextlib.nullcontext()):
                if scoped:
                    fork.wait()
                for i in range(w, len(items), k):
                    out[i] = fn(items[i])
                if scoped:
                    done[w].record()
        except BaseException as e:  # surfaced on the caller's thread
            errs.append(e)

    th = [threading.Thread(target=worker, args=(w,)) for w in range(k)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    if scoped:
        for e in done:
            e.wait()  # the caller's stream continues after every worker's work
    return out


# ---------------------------------------------------------------------------
# Config 2: encrypted linear score (pt x ct multiply-accumulate)
# ---------------------------------------------------------------------------

ATTR_NORM = 8 * 255.0  # folds the [0,255] attribute range and the 8-term sum into [-1, 1]


def linear_score_data(spec: Spec, seed_offset: int = 0):
    """Server records (8 integer attributes in [0,255]) and the scientist's
    weights w_j ~ U[-1,1]."""
    g = np.random.Generator(np.random.PCG64(spec.seed + seed_offset))
    attrs = g.integers(0, 256, size=(spec.records, 8)).astype(np.float64)
    w = g.uniform(-1.0, 1.0, size=8)
    return attrs, w


def encode_plaintexts(S, columns, level, to_eval=True):
    """Server-side plaintexts: each row of `columns` (a slot vector) encoded at
    scale q_level (the mul_scalar convention, so a following rescale restores
    the ciphertext scale) and transformed to eval form for mul_plain
    (ckks.hpp:253-269). The B200 module encodes the batch in one device launch."""
    scale = float(S.ring.modulus(level))
    arr = np.asarray(columns, dtype=np.complex128).reshape(-1, S.spec.slots)
    pts = S.encode(S, arr, scale, level)
    if to_eval:
        for p in pts:
            p.ntt_forward()
    return pts, scale


def encrypt_many(S, vectors, level, labels):
    """Scientist-side encryption (KeyContext::encrypt, secret key) of slot
    vectors at scale Delta, randomness Rng(seed).split(label)."""
    T = S.T
    arr = np.asarray(vectors, dtype=np.complex128).reshape(-1, S.spec.slots)
    ms = S.encode(S, arr, S.spec.delta, level)
    return [S.ctx.encrypt(S.sk, m, S.spec.delta, T.Rng(S.spec.seed).split(lab), T.Domain.slots)
            for m, lab in zip(ms, labels)]


def weights_eval(S, ct_w):
    """B200 module: the query's 8 weight ciphertexts -- shared by every record
    block's linear score -- forward-transformed ONCE per query as one stacked
    batch (one batched NTT; mul_plain_sum reads the batch's part-major views
    in place). Otherwise (or with a single weight) unchanged: per-ciphertext
    to_eval inside mul_plain_sum, memoised on the first block."""
    T = S.T
    ct_w = list(ct_w)
    if not hasattr(T, "stack_ciphertexts") or len(ct_w) < 2 or os.environ.get("TG_WEIGHTS_EVAL") == "0":
        return ct_w
    st = T.stack_ciphertexts(ct_w)
    st.to_eval()
    return T.unstack_ciphertext(st)


def linear_score(S, ct_w, pts, plain_scale):
    """score = rescale(sum_j mul_plain(ct_w_j, pt_j)), summed in j order
    (config 2's pt x ct MAC)."""
    ev = S.ev
    if hasattr(ev, "mul_plain_sum"):  # B200 module: the 8 products and 7 adds in one pass
        return ev.rescale(ev.mul_plain_sum(list(ct_w), list(pts), plain_scale))
    acc = None
    for cw, p in zip(ct_w, pts):
        t = ev.mul_plain(cw, p, plain_scale)
        acc = t if acc is None else ev.add(acc, t)
    return ev.rescale(acc)


def config2_inputs(S, attrs=None, w=None):
    spec = S.spec
    if attrs is None:
        attrs, w = linear_score_data(spec)
    n, L = spec.slots, S.ring.max_level()
    ct_w = encrypt_many(S, [[wj] * n for wj in w], L, [400 + j for j in range(8)])
    cols = [attrs[b * n:(b + 1) * n, j] / ATTR_NORM for b in range(spec.n_cts) for j in range(8)]
    pts, pscale = encode_plaintexts(S, cols, L)
    blocks = [pts[8 * b:8 * b + 8] for b in range(spec.n_cts)]
    return SimpleNamespace(ct_w=ct_w, blocks=blocks, plain_scale=pscale, attrs=attrs, w=w)


def config2_query(S, inp, streams=1):
    ct_w = weights_eval(S, inp.ct_w)
    return run_concurrent(S.T, S.ring, lambda pts: linear_score(S, ct_w, pts, inp.plain_scale),
                          inp.blocks, streams)


# ---------------------------------------------------------------------------
# Configs 4-5: the full TETRIS statement
# ---------------------------------------------------------------------------

RISK_NORM = 0.5  # |risk - t| <= 1.05 for risk in [-1,1], |t| <= 0.05
COLUMNS = ("risk", "sugar", "bp")   # threshold job columns, in upload order
COLUMN_T = {"risk": 2, "sugar": 0, "bp": 1}  # index into the query's thresholds
COLUMN_NORM = {"risk": RISK_NORM, "sugar": 1.0, "bp": 1.0}


def statement_data(spec: Spec, seed_offset: int = 0):
    """Synthetic records with BASELINE.json's distributions, each attribute
    normalised by its clip range, plus the scientist's statement:
    sugar >= 126 mg/dL AND pressure >= 140 mmHg AND risk >= t_risk AND flag."""
    g = np.random.Generator(np.random.PCG64(spec.seed + seed_offset))
    n = spec.records
    sugar = np.clip(g.normal(100.0, 25.0, n), 40.0, 300.0)
    bp = np.clip(g.normal(120.0, 15.0, n), 70.0, 220.0)
    flag = (g.random(n) < 0.1).astype(np.float64)
    attrs = g.integers(0, 256, size=(n, 8)).astype(np.float64)
    w = g.uniform(-1.0, 1.0, size=8)
    t = ((126.0 - 40.0) / 260.0, (140.0 - 70.0) / 150.0, float(g.uniform(-0.05, 0.05)))
    return SimpleNamespace(sugar=(sugar - 40.0) / 260.0, bp=(bp - 70.0) / 150.0, flag=flag,
                           attrs=attrs / ATTR_NORM, w=w, t=t)


def statement_plain_count(d):
    """Plaintext comparator (informational; the exact check is against the
    oracle's decrypted count, SURVEY 8(d) config 3 note)."""
    risk = d.attrs @ d.w
    return int(((d.sugar >= d.t[0]) & (d.bp >= d.t[1]) & (risk >= d.t[2]) & (d.flag > 0)).sum())


def statement_query_inputs(S, d):
    """The scientist's encrypted statement: 8 risk weights and 3 thresholds."""
    n, L = S.spec.slots, S.ring.max_level()
    vecs = [[wj] * n for wj in d.w] + [[tk] * n for tk in d.t]
    cts = encrypt_many(S, vecs, L, [400 + j for j in range(8)] + [90, 91, 92])
    return SimpleNamespace(ct_w=cts[:8], ct_t=cts[8:])


def statement_block_inputs(S, d, b):
    """Record block b: encrypted sugar/pressure columns, plaintext risk
    attributes and plaintext flag (eval form, level L, scale q_L). The flag
    multiplies the AND output, whose level depends on the polynomial
    evaluator (BSGS saves a level on degree 27); a level-L plaintext serves
    any level (mul_plain reads rows by modulus index, ckks.hpp:257-265), and
    the tracked scale absorbs q_L / q_level after the rescale."""
    n = S.spec.slots
    L = S.ring.max_level()
    sl = slice(b * n, (b + 1) * n)
    cts = encrypt_many(S, [d.sugar[sl], d.bp[sl]], L, [200 + b, 300 + b])
    pts, ascale = encode_plaintexts(S, [d.attrs[sl, j] for j in range(8)] + [d.flag[sl]], L)
    flag, fscale = pts[8:], ascale
    pts = pts[:8]
    return SimpleNamespace(ct_sugar=cts[0], ct_bp=cts[1], pt_attr=pts, attr_scale=ascale,
                           pt_flag=flag[0], flag_scale=fscale)


def mul_relin_rescale(ev, a, b, keys):
    """rescale(mul_relin(a, b)); one ModDown + rescale pass where the evaluator
    has it (Evaluator::mul_relin_rescale, identical residues and metadata)."""
    f = getattr(ev, "mul_relin_rescale", None)
    return f(a, b, keys) if f is not None else ev.rescale(ev.mul_relin(a, b, keys))


def statement_block(S, q, blk, threshold):
    """One block of the statement in the reference API's op order:
    linear risk score, three private thresholds (threshold(x, t, norm)),
    AND = rescale(mul_relin(b1, b2)) then x b3, then the flag product."""
    ev, keys = S.ev, S.keys
    risk = linear_score(S, q.ct_w, blk.pt_attr, blk.attr_scale)
    b1 = threshold(blk.ct_sugar, q.ct_t[0], 1.0)
    b2 = threshold(blk.ct_bp, q.ct_t[1], 1.0)
    b3 = threshold(risk, q.ct_t[2], RISK_NORM)
    a = ev.rescale(ev.mul_relin(b1, b2, keys))
    a = ev.rescale(ev.mul_relin(a, b3, keys))
    return ev.rescale(ev.mul_plain(a, blk.pt_flag, blk.flag_scale))


def threshold_fn(S, chain, mode=None):
    T = S.T
    if mode is None:
        return lambda x, t, norm: T.eval_private_threshold_plain_norm(S.ev, x, t, norm, chain, S.keys)
    return lambda x, t, norm: T.eval_private_threshold_plain_norm(S.ev, x, t, norm, chain, S.keys, mode)


def statement_partial(S, q, blocks, threshold, streams=1):
    """Sum (mod q, block order) of the per-block statements on this shard."""
    outs = run_concurrent(S.T, S.ring, lambda blk: statement_block(S, q, blk, threshold), blocks, streams)
    acc = None
    for o in outs:
        acc = o if acc is None else S.ev.add(acc, o)
    return acc


def statement_jobs(nblocks: int, max_batch: int):
    """The (column, block) threshold jobs of `nblocks` record blocks cut into
    ciphertext batches of <= max_batch near-equal parts: the risk column
    (its inputs are resident first in a staged upload; level L-1 after the
    score's rescale, norm RISK_NORM) on its own, the sugar and pressure
    columns (level L, norm 1) together, so a batch may mix those two and a
    shard of one record block still runs them as one batch of two."""
    out = []
    for group in (("risk",), ("sugar", "bp")):
        jobs = [(col, i) for col in group for i in range(nblocks)]
        if not jobs:
            continue
        nb = -(-len(jobs) // max(1, max_batch))
        size = -(-len(jobs) // nb)
        out += [jobs[i:i + size] for i in range(0, len(jobs), size)]
    return out


def statement_partial_batched(S, q, blocks, threshold, streams=2, max_blocks=8, ready=None, keep=None):
    """B200 module: the per-block statement with the blocks evaluated as
    ciphertext batches (stack_ciphertexts): the (column, block) threshold jobs
    in batches of <= max_blocks (statement_jobs; the batches run on
    concurrent streams), then the AND products per chunk of <= max_blocks
    blocks, batched. Each block's output is bit-identical to
    statement_block's (a batch is exactly `batch` independent ciphertexts;
    tests/test_gpu_statement.py); launches and switching-key reads are shared
    by the batch.
    ready (optional, staged uploads): ready(name) makes the current stream
    wait until the client ciphertexts `name` ("w", "t0".."t2", "sugar", "bp") are
    resident, so each job starts as soon as its own inputs have arrived.
    keep (optional list): receives every block's output before the sum."""
    T, ev, keys = S.T, S.ev, S.keys
    wait = ready or (lambda name: None)
    wait("w")
    ct_w = weights_eval(S, q.ct_w)

    def score(blk):
        return linear_score(S, ct_w, blk.pt_attr, blk.attr_scale)

    risks = run_concurrent(T, S.ring, score, blocks, streams)
    batches = statement_jobs(len(blocks), max_blocks)

    def job(batch):
        xs, ts = [], []
        for col, i in batch:
            k = COLUMN_T[col]
            wait(f"t{k}")  # this job's threshold only
            if col != "risk":
                wait(col)
            xs.append(risks[i] if col == "risk" else getattr(blocks[i], "ct_" + col))
            ts.append(q.ct_t[k])
        return threshold(T.stack_ciphertexts(xs), T.stack_ciphertexts(ts), COLUMN_NORM[batch[0][0]])

    outs = run_concurrent(T, S.ring, job, batches, streams)
    where = {}  # (column, block) -> (batch, position)
    for bi, batch in enumerate(batches):
        for pos, jb in enumerate(batch):
            where[jb] = (bi, pos)
    pieces = {}

    def indicator(col, i):
        bi, pos = where[(col, i)]
        if outs[bi].batch == 1:
            return outs[bi]
        if bi not in pieces:
            pieces[bi] = T.unstack_ciphertext(outs[bi])
        return pieces[bi][pos]

    def column_batch(col, chunk):
        """The indicators of `col` for the blocks of `chunk` as one batch: a
        job batch as it is when it holds exactly those, else restacked."""
        bi, _ = where[(col, chunk[0])]
        if batches[bi] == [(col, i) for i in chunk]:
            return outs[bi]
        xs = [indicator(col, i) for i in chunk]
        return xs[0] if len(xs) == 1 else T.stack_ciphertexts(xs)

    acc = None
    for c0 in range(0, len(blocks), max_blocks):
        chunk = list(range(c0, min(len(blocks), c0 + max_blocks)))
        b1, b2, b3 = column_batch("sugar", chunk), column_batch("bp", chunk), column_batch("risk", chunk)
        a = mul_relin_rescale(ev, b1, b2, keys)
        a = mul_relin_rescale(ev, a, b3, keys)
        for i, ct in zip(chunk, T.unstack_ciphertext(a) if a.batch > 1 else [a]):
            o = ev.rescale(ev.mul_plain(ct, blocks[i].pt_flag, blocks[i].flag_scale))
            if keep is not None:
                keep.append(o)
            acc = o if acc is None else ev.add(acc, o)
    return acc
