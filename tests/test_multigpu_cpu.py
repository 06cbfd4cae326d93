"""Multi-rank exchange of the threshold-count query on CPU (gloo, world size
2 and 3): sharding covers every ciphertext exactly once, and the integer
SUM-reduce of partial ciphertexts + mod-q fix-up equals the sequential
mod-q sum (Ciphertext::add_inplace, rlwe.hpp:300-305) bit for bit — the
property that makes the multi-GPU count identical to the single-GPU one."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_13269_b200 import distributed as D

N = 1024
MODULI = [1125899906826241, 1125899906629633, 1125899906727937, 1152921504606830593]  # 3 x ~50-bit, 1 x 60-bit


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _partial(rank):
    rng = np.random.default_rng(1000 + rank)
    return np.stack([rng.integers(0, q, size=N, dtype=np.uint64) for q in MODULI])


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        part = _partial(rank)
        t = torch.from_numpy(part.view(np.int64).copy())
        D.reduce_to_root(dist, [t])
        if rank == 0:
            out_q.put(D.fixup_mod_q_host(t.numpy().view(np.uint64), MODULI))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_integer_reduce_equals_modq_sum(world):
    D.check_exact(world, MODULI)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = _partial(0)
    for r in range(1, world):
        nxt = _partial(r)
        for row, qm in enumerate(MODULI):
            s = want[row] + nxt[row]  # < 2^64: add_mod semantics (common.hpp:24-27)
            want[row] = np.where(s >= np.uint64(qm), s - np.uint64(qm), s)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n_items,world", [(4, 1), (4, 2), (4, 8), (8, 3), (32, 8)])
def test_shard_partition(n_items, world):
    seen = sorted(b for r in range(world) for b in D.shard(n_items, world, r))
    assert seen == list(range(n_items))


def test_exactness_guard():
    with pytest.raises(ValueError):
        D.check_exact(32, [1 << 62])


# ---------------------------------------------------------------------------
# The bench's multi-GPU algorithm end to end, with the reference module (CPU)
# doing the ring arithmetic: round-robin shards of record blocks, per-rank
# statement partial sums, integer SUM-reduce to rank 0 (gloo here, NCCL on
# GPUs), mod-q fix-up, one inner_sum on rank 0 == the single-process count.
# ---------------------------------------------------------------------------
def _statement_setup():
    import dataclasses
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from common import load_ref
    from paper_2412_13269_b200 import workloads as W
    R = load_ref()
    spec = dataclasses.replace(W.CONFIGS[4], N=256, records=3 * 128, n_cts=3)
    S = W.make_context(R, spec, rotations=W.inner_sum_rotations(spec.slots))
    chain = W.config3_chain(R, spec)
    d = W.statement_data(spec)
    d.t = (0.2, 0.3, -0.02)
    q = W.statement_query_inputs(S, d)
    return R, W, spec, S, chain, d, q


def _statement_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        R, W, spec, S, chain, d, q = _statement_setup()
        mine = D.shard(spec.n_cts, world, rank)
        blocks = [W.statement_block_inputs(S, d, b) for b in mine]
        acc = W.statement_partial(S, q, blocks, W.threshold_fn(S, chain)) if blocks else None
        lv = torch.tensor([acc.level() if acc is not None else -1], dtype=torch.int64)
        dist.all_reduce(lv, op=dist.ReduceOp.MAX)  # ranks without blocks learn the output level
        if acc is None:
            acc = S.ctx.zero_ciphertext(int(lv.item()), 1.0, S.sk.id(), R.Domain.slots)
        parts = [torch.from_numpy(p.to_numpy().view(np.int64).copy()) for p in acc.parts]
        D.reduce_to_root(dist, parts)
        if rank == 0:
            moduli = [S.ring.modulus(i) for i in range(acc.level() + 1)]
            ct = R.Ciphertext()
            ct.parts = [R.Poly.from_numpy(S.ring, D.fixup_mod_q_host(t.numpy().view(np.uint64), moduli),
                                          acc.level(), acc.form(), 0) for t in parts]
            ct.scale, ct.domain, ct.sk_id = acc.scale, acc.domain, acc.sk_id
            count = R.inner_sum(S.ev, ct, spec.slots, S.keys)
            out_q.put([p.to_numpy() for p in count.parts] + [count.scale, count.level()])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_statement_count_bit_exact(world):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from common import load_ref
    if load_ref() is None:
        pytest.skip("oracle/_ref not built")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_statement_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # single process, all blocks, the reference order (sum, then one inner_sum)
    R, W, spec, S, chain, d, qi = _statement_setup()
    blocks = [W.statement_block_inputs(S, d, b) for b in range(spec.n_cts)]
    want = R.inner_sum(S.ev, W.statement_partial(S, qi, blocks, W.threshold_fn(S, chain)), spec.slots, S.keys)
    assert got[-1] == want.level() and got[-2] == want.scale
    for a, b in zip(got[:-2], want.parts):
        assert np.array_equal(a, b.to_numpy())


@pytest.mark.parametrize("n_blocks,world", [(8, 1), (8, 2), (8, 4), (8, 8), (32, 8), (3, 2)])
def test_statement_jobs_keep_batches_under_sharding(n_blocks, world):
    """Every rank's (column, block) threshold jobs are covered exactly once,
    batches never mix levels (the risk column runs one level lower after the
    score's rescale), and a rank with one record block still runs its sugar
    and pressure thresholds as ONE batch of two (batching must
    survive sharding at 8 GPUs)."""
    from paper_2412_13269_b200 import workloads as W
    for rank in range(world):
        mine = D.shard(n_blocks, world, rank)
        batches = W.statement_jobs(len(mine), 8)
        jobs = [j for b in batches for j in b]
        assert sorted(jobs) == sorted((c, i) for c in W.COLUMNS for i in range(len(mine)))
        for b in batches:
            assert len(b) <= 8
            assert len({c == "risk" for c, _ in b}) == 1  # one level per batch
            assert len({W.COLUMN_NORM[c] for c, _ in b}) == 1
        if mine:
            sb = [b for b in batches if b[0][0] != "risk"]
            assert min(len(b) for b in sb) >= min(2, 2 * len(mine))
