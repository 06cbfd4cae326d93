"""Full-size parity of the path bench.py times (VERDICT r1 top
item): BSGS polynomial evaluation with record blocks stacked as ciphertext
batches, at the configs' own N = 2^16 rings, chains and gadgets, against the
BSGS oracle (oracle/bsgs_ref.py over the compiled reference oracle/_ref).

  config 3: the whole query (4 score blocks as one batch of 4, sum, one
            inner_sum) == the oracle's, residue for residue, and the same
            decrypted count (threshold.hpp:146-157, protocol.hpp:319-323).
  config 4: all 8 record blocks through the batched statement (three
            batches of 8 threshold jobs, batched AND); blocks 0 and 7 ==
            the oracle's per-block statement, and the count of their
            sum + inner_sum is identical.
"""
import dataclasses
import os
import sys
from pathlib import Path

import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402  (the bench's own workload drivers: the shipped path)
import fullsize as F  # noqa: E402
from paper_2412_13269_b200 import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu


def _threads(n):
    return max(1, min(n, os.cpu_count() or 1))


def test_config3_full_query_bit_exact(G, R, gpu_available):
    spec = W.CONFIGS[3]
    wl = bench.ThresholdCount(G, W, spec)
    secs, nb, chk = wl.oracle_check(R, W, _threads(spec.n_cts))
    assert chk["bit_exact_vs_oracle_bsgs"], chk
    assert round(chk["gpu_decrypted_count"]) == round(chk["oracle_decrypted_count"])
    assert abs(chk["gpu_decrypted_count"] - chk["oracle_decrypted_count"]) < 2.0 ** -20 * spec.records


def test_config4_blocks_0_and_7_bit_exact(G, R, gpu_available):
    spec = W.CONFIGS[4]
    wl = bench.Statement(G, W, spec)
    assert wl.max_blocks == 8 and len(wl.blocks) == 8  # the shipped batching
    secs, nb, chk = wl.oracle_check(R, W, _threads(6))
    assert chk["oracle_blocks"][0] == 0 and chk["oracle_blocks"][-1] == 7
    assert chk["bit_exact_vs_oracle_bsgs"], chk
    assert round(chk["gpu_decrypted_count"]) == round(chk["oracle_decrypted_count"])


def test_statement_one_block_shard_mixed_batch(G, R, gpu_available):
    """A rank holding ONE record block (8 GPUs, config 4): its sugar and
    pressure thresholds run as one mixed batch of two (statement_jobs), and
    the block's output still equals the oracle's."""
    spec = dataclasses.replace(W.CONFIGS[4], N=1 << 12, records=1 << 11, n_cts=1)
    assert W.statement_jobs(1, 8) == [[("risk", 0)], [("sugar", 0), ("bp", 0)]]
    wl = bench.Statement(G, W, spec)
    secs, nb, chk = wl.oracle_check(R, W, 3)
    assert chk["bit_exact_vs_oracle_bsgs"], chk
