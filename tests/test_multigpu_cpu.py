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
