"""Multi-GPU exchange of the threshold-count query.

Ciphertext blocks shard round-robin over ranks; each rank sums its
per-ciphertext threshold outputs mod q; the partial ciphertexts are reduced
to rank 0 with an integer SUM (NCCL on GPUs, gloo in the CPU tests) and rank 0
restores canonical residues mod q (tg_poly_reduce on the device) before the
single inner_sum — the reference order (protocol.hpp:319-323), so the result
is bit-identical for every world size.

Exactness: every word is < q_max < 2^62 and world * q_max < 2^64 (checked), so
the wrapped int64 sum equals the exact integer sum of the residues.
"""
from __future__ import annotations

from typing import Sequence


def shard(n_items: int, world: int, rank: int) -> list[int]:
    """Round-robin assignment of ciphertext blocks to ranks."""
    return [b for b in range(n_items) if b % world == rank]


def check_exact(world: int, moduli: Sequence[int]) -> None:
    if world * max(int(q) for q in moduli) >= 1 << 64:
        raise ValueError("integer reduce not exact: world * q_max >= 2^64")


def reduce_to_root(dist, tensors, group=None) -> None:
    """In-place integer SUM of each tensor (int64 views of u64 words) into rank 0."""
    for t in tensors:
        dist.reduce(t, dst=0, op=dist.ReduceOp.SUM, group=group)


def fixup_mod_q_host(words, row_moduli):
    """Host mirror of tg_poly_reduce for the CPU tests: words (rows, N) as
    uint64 holding exact integer sums -> canonical residues per row."""
    import numpy as np

    out = np.empty_like(words)
    for r, q in enumerate(row_moduli):
        out[r] = words[r] % np.uint64(q)
    return out
