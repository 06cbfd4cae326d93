#!/usr/bin/env python3
"""Benchmark of the B200 RNS-CKKS TETRIS query (BASELINE.json metric:
encrypted records/s & amortized us/record per TETRIS query).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--config 4|3|5] [--poly-eval bsgs|ladder] [--streams S]

Default workload: config 4, the full TETRIS statement over 2^18 records
(N=2^16, L=21): per record block (2^15 records per ciphertext) an encrypted
8-attribute linear risk score (8 pt x ct MACs + rescale), three private
thresholds (composite minimax sign chain (15,15,27), BSGS), the AND as
products of indicators, the plaintext disorder flag, the sum over blocks and
the log2(slots) rotate-and-add slot sum into one encrypted count.
Config 3 (threshold count, 2^17 records) and config 5 (2^20 records,
degree-63 chain, L=28, dnum=3) run with --config.

One step = one full query. N>1 (torchrun): record blocks are sharded
round-robin over ranks; each rank sums its block outputs, the partial
ciphertexts are NCCL-reduced to rank 0 (integer sum + mod-q fix-up kernel)
and rank 0 runs the one inner_sum - the reference's order (sum, then
InnerSum; protocol.hpp:319-323), so the count is bit-identical at every GPU
count.

`--impl reference` times the reference's own CPU implementation (the
unmodified headers compiled into oracle/_ref) on the box's host cores with
threads over blocks and thresholds (protocol.hpp:297-311); rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, os.environ.get("TG_ROOT", str(ROOT)))  # TG_ROOT: a variant build (tools/build_variant.sh)

RECORDS_PER_CT = None  # set from the spec


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md: sample during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock + clock-event reasons sampled in-process through NVML every
    0.1 s during the timed region (spawning nvidia-smi repeatedly stalls the
    driver and shows up as step-time spikes)."""
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))

    def __init__(self, device: int, pci_bus_id: str | None = None):
        self.device = device
        self.pci = pci_bus_id
        self.samples: list[tuple[int, int, int]] = []
        self._stop = threading.Event()
        self._thr = None
        self.error = None

    def _run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            try:
                h = pynvml.nvmlDeviceGetHandleByPciBusId(self.pci) if self.pci else None
            except Exception:
                h = None
            if h is None:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                try:
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                except Exception:
                    rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append((sm, smax, rs))
                self._stop.wait(0.1)
            pynvml.nvmlShutdown()
        except Exception as e:  # reported in the JSON line
            self.error = str(e)[:120]

    def __enter__(self):
        if os.environ.get("TG_NO_CLOCKS") == "1":  # diagnostics: no sampler
            return self
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thr:
            self._thr.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.error or "NVML unavailable"],
                    "samples": 0}
        reasons = sorted({n for _, _, rs in self.samples for n, bit in self.REASONS if rs & bit})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": "NVML"}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class _CAI:
    """__cuda_array_interface__ view of a device buffer (zero copy)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<u8", "data": (ptr, False), "version": 3,
                                         "strides": None}


FP64_PEAK_OPS = 18.3e12  # DP ops/s, tools/diag/fp64_peak.cu on this pool's B200 (61-63 ops/clk/SM at 1965 MHz)


def fp64_roofline_class(prof, name):
    """FP64-pipe roofline of one kernel class whose algorithmic FP64 op count
    the profiler records (tg_profile_read_ops: the fused key-switch core, 8 ops
    per chunk-phase butterfly and 7 per key-inner-product term) against the
    measured FP64 peak; None when not modelled."""
    v = prof.get(name)
    if not v or len(v) < 4 or v[3] <= 0 or v[0] <= 0:
        return None
    ach = v[3] / (v[0] / 1e3)
    return {"kernel": name, "achieved": round(ach / 1e12, 3), "peak": FP64_PEAK_OPS / 1e12,
            "unit": "TFLOP/s (FP64 DP ops, algorithmic: 8 per butterfly, 7 per key MAC term)",
            "frac": round(ach / FP64_PEAK_OPS, 4), "ops_per_launch": v[3] / v[1],
            "peak_kind": "measured (tools/diag/fp64_peak.cu: DADD/DMUL/DFMA throughput probe)"}


def fp64_roofline(prof, N):
    """FP64-pipe roofline of the NTT classes: algorithmic ops (8 per
    butterfly) per second vs the measured FP64 peak."""
    import math
    ms = sum(v[0] for k, v in prof.items() if k.startswith("ntt"))
    byts = sum(v[2] for k, v in prof.items() if k.startswith("ntt"))
    if ms <= 0:
        return None
    ops = byts * math.log2(N) / 4.0
    ach = ops / (ms / 1e3)
    return {"kernel": "ntt (fwd+inv)", "achieved": round(ach / 1e12, 3), "peak": FP64_PEAK_OPS / 1e12,
            "unit": "TFLOP/s (FP64 DP ops, 8 per butterfly)", "frac": round(ach / FP64_PEAK_OPS, 4),
            "peak_kind": "measured (tools/diag/fp64_peak.cu: DADD/DMUL/DFMA throughput probe)"}


def reduce_partial_to_root(G, torch, dist, ct, ext_stream, N):
    """Integer NCCL sum of every rank's partial ciphertext into rank 0's
    buffer (exact: ranks * q < 2^64 for the <=60-bit q-chain), then the mod-q
    fix-up kernel on rank 0. Stream-ordered, no host sync."""
    ready = torch.cuda.Event()
    ready.record(ext_stream)
    cur = torch.cuda.current_stream()
    cur.wait_event(ready)
    n = ct.parts[0].rows() * N
    for p in ct.parts:
        t = torch.as_tensor(_CAI(p.device_ptr(), n), device="cuda").view(torch.int64)
        dist.reduce(t, dst=0, op=dist.ReduceOp.SUM)
    done = torch.cuda.Event()
    done.record(cur)
    ext_stream.wait_event(done)
    if dist.get_rank() == 0:
        G.ciphertext_reduce_inplace(ct)


# ---------------------------------------------------------------------------
# Workloads: per-query client ciphertexts (uploaded by the e2e leg), resident
# server data, and the per-rank partial result before the NCCL reduce.
# ---------------------------------------------------------------------------
def decrypted_count(G, S, spec, res, plain):
    enc = G.Encoder(S.ring, spec.slots)
    dec = np.array(enc.decode_slots(S.ctx.decrypt(S.sk, res), res.scale))
    return {"decrypted_count": round(float(dec[0].real), 3), "plaintext_comparator_count": plain,
            "count_level": res.level()}


def _timed_encode(SR, arr, scale, level, threads):
    """The reference's own Encoder::encode_slots over every row of `arr`
    (oracle/_ref binding: the unmodified code on a std::thread pool)."""
    enc = SR.T.Encoder(SR.ring, SR.spec.slots)
    return list(enc.encode_slots_many(np.asarray(arr, dtype=np.complex128), scale, level, threads))


class ThresholdCount:
    """Config 3: private threshold of every encrypted score block against an
    encrypted threshold (plain norm), summed."""
    metric = "encrypted records/sec per TETRIS threshold-count query (amortized us/record in config)"
    slot_sum = True
    columns = 1  # threshold jobs per record block

    def check(self, res):
        return decrypted_count(self.G, self.S, self.spec, res, self.plain_count())

    def __init__(self, G, W, spec, rank=0, world=1, rotations=True, device=True):
        self.G, self.W, self.spec = G, W, spec
        self.batched, self.max_blocks = True, 8
        self.scores, self.thr, _, _ = W.linear_scores(spec)
        if not device:  # inputs only (the CPU reference arm: no product import)
            return
        from paper_2412_13269_b200 import distributed as D
        rot = W.inner_sum_rotations(spec.slots) if rotations else []
        self.S = W.make_context(G, spec, rotations=rot)
        self.chain = W.config3_chain(G, spec)
        self.mine = D.shard(spec.n_cts, world, rank)
        cts, ct_t, _, _ = W.config3_inputs(self.S, ct_indices=self.mine, scores=self.scores, t=self.thr)
        self.client = cts + [ct_t]

    def partial(self, client, streams, mode, keep=None):
        cts, ct_t = client[:-1], client[-1]
        if not cts:
            return None
        if self.batched and len(cts) > 1:  # all score blocks as one ciphertext batch
            G, ev = self.G, self.S.ev
            fat = G.eval_private_threshold_plain_norm(ev, G.stack_ciphertexts(cts),
                                                     G.stack_ciphertexts([ct_t] * len(cts)), self.spec.norm,
                                                     self.chain, self.S.keys, mode)
            outs = G.unstack_ciphertext(fat)
        else:
            outs = self.G.eval_private_threshold_plain_norm_many(self.S.ev, cts, ct_t, self.spec.norm, self.chain,
                                                                 self.S.keys, streams, mode)
        if keep is not None:
            keep.extend(outs)
        acc = outs[0]
        for o in outs[1:]:
            acc = self.S.ev.add(acc, o)
        return acc

    def plain_count(self):
        return int((self.scores >= self.thr).sum())

    def ref_inputs(self, SR, blocks, threads):
        """Client ciphertexts of `blocks` for the reference arm, encoded by the
        reference's own Encoder (threaded) and encrypted with the same Rng
        labels as the B200 arm's (bit-identical inputs)."""
        W, n, L = self.W, self.spec.slots, SR.ring.max_level()
        vecs = [self.scores[b * n:(b + 1) * n] for b in blocks] + [[self.thr] * n]
        t0 = time.perf_counter()
        ms = _timed_encode(SR, vecs, self.spec.delta, L, threads)
        enc_s = time.perf_counter() - t0
        labels = [100 + b for b in blocks] + [99]
        cts = [SR.ctx.encrypt(SR.sk, m, self.spec.delta, SR.T.Rng(self.spec.seed).split(lab), SR.T.Domain.slots)
               for m, lab in zip(ms, labels)]
        return (cts[:-1], cts[-1]), {"client_vectors": len(vecs), "client_encode_s": round(enc_s, 2),
                                     "server_vectors": 0, "server_encode_s": 0.0}

    def ref_step(self, R, SR, chain_r, inp, threads):
        """The reference's own threshold on every block (thread pool,
        protocol.hpp:297-311), sum in block order, one inner_sum. Returns
        (count ciphertext, {phase: seconds})."""
        cts, ct_t = inp
        t0 = time.perf_counter()
        acc = R.threshold_count_pool(SR.ev, cts, ct_t, self.spec.norm, chain_r, SR.keys, self.spec.slots,
                                     threads, False)[0]
        t1 = time.perf_counter()
        cnt = R.inner_sum(SR.ev, acc, self.spec.slots, SR.keys)
        return cnt, {"blocks_s": t1 - t0, "slot_sum_s": time.perf_counter() - t1}

    def oracle_check(self, R, W, threads):
        """Full query through the BSGS oracle (all blocks + inner_sum) vs the
        product's full query output, residue for residue and by count."""
        import fullsize as F
        SR, chain_r = F.oracle_context(R, W, self.spec, self.S, self.chain)
        cnt_r, outs_r, secs = F.oracle_threshold_count(R, W, SR, chain_r, self.scores, self.thr,
                                                       list(range(self.spec.n_cts)), threads)
        keep = []
        acc = self.partial(self.client, 4, self.G.PolyEval.bsgs, keep=keep)
        cnt_g = self.G.inner_sum(self.S.ev, acc, self.spec.slots, self.S.keys)
        same_blocks = all(F.ct_equal(a, b) for a, b in zip(keep, outs_r))
        return secs, len(outs_r), {
            "oracle_blocks": list(range(self.spec.n_cts)),
            "bit_exact_vs_oracle_bsgs": bool(same_blocks and F.ct_equal(cnt_g, cnt_r)),
            "oracle_decrypted_count": round(F.decrypted_count(SR, cnt_r), 3),
            "gpu_decrypted_count": round(F.decrypted_count(self.S, cnt_g), 3),
            "what": "the whole query (all score blocks, sum, inner_sum) through the product path as timed vs the "
                    "BSGS oracle (oracle/bsgs_ref.py over oracle/_ref)"}


class Statement:
    """Configs 4/5: the full TETRIS statement per record block (linear risk
    score, three private thresholds, AND, plaintext flag), summed."""
    metric = "encrypted records/sec per TETRIS query (full statement; amortized us/record in config)"
    slot_sum = True
    columns = 3

    def check(self, res):
        return decrypted_count(self.G, self.S, self.spec, res, self.plain_count())

    def __init__(self, G, W, spec, rank=0, world=1, rotations=True, device=True):
        self.G, self.W, self.spec = G, W, spec
        self.batched, self.max_blocks = True, 8
        self.d = W.statement_data(spec)
        if not device:  # inputs only (the CPU reference arm: no product import)
            return
        from paper_2412_13269_b200 import distributed as D
        rot = W.inner_sum_rotations(spec.slots) if rotations else []
        self.S = W.make_context(G, spec, rotations=rot)
        self.chain = W.config3_chain(G, spec)
        self.mine = D.shard(spec.n_cts, world, rank)
        q = W.statement_query_inputs(self.S, self.d)
        self.blocks = [W.statement_block_inputs(self.S, self.d, b) for b in self.mine]
        # client ciphertexts in the order the query consumes them (staged
        # uploads, e2e): each threshold job needs its column and ONE threshold,
        # so the first job (risk: weights + t2) starts after 198 MB, not after
        # all three thresholds as well
        nb = len(self.blocks)
        self.client = (q.ct_w + [q.ct_t[2], q.ct_t[0]] + [b.ct_sugar for b in self.blocks] + [q.ct_t[1]] +
                       [b.ct_bp for b in self.blocks])
        self.upload_groups = {"w": (0, 8), "t2": (8, 9), "t0": (9, 10), "sugar": (10, 10 + nb),
                              "t1": (10 + nb, 11 + nb), "bp": (11 + nb, 11 + 2 * nb)}

    def _bind(self, client, blocks):
        from types import SimpleNamespace as NS
        nb = len(blocks)
        q = NS(ct_w=client[:8], ct_t=[client[9], client[10 + nb], client[8]])
        bl = [NS(ct_sugar=client[10 + i], ct_bp=client[11 + nb + i], pt_attr=b.pt_attr,
                 attr_scale=b.attr_scale, pt_flag=b.pt_flag, flag_scale=b.flag_scale)
              for i, b in enumerate(blocks)]
        return q, bl

    def partial(self, client, streams, mode, ready=None, keep=None):
        if not self.blocks:
            return None
        q, bl = self._bind(client, self.blocks)
        thr = self.W.threshold_fn(self.S, self.chain, mode)
        if self.batched:  # (column, block) jobs as ciphertext batches (shared launches and key reads)
            return self.W.statement_partial_batched(self.S, q, bl, thr, streams=streams, max_blocks=self.max_blocks,
                                                    ready=ready, keep=keep)
        if ready:
            for name in self.upload_groups:
                ready(name)
        return self.W.statement_partial(self.S, q, bl, thr, streams)

    def plain_count(self):
        return self.W.statement_plain_count(self.d)

    def server_plaintexts(self, S, blocks):
        """Server-side plaintexts of `blocks` (8 risk attributes + the flag
        per block): the slot vectors encoded at scale q_L and NTT'd."""
        n = self.spec.slots
        return [self.d.attrs[b * n:(b + 1) * n, j] for b in blocks for j in range(8)] + \
               [self.d.flag[b * n:(b + 1) * n] for b in blocks]

    def ref_inputs(self, SR, blocks, threads):
        """The query's and `blocks`' inputs for the reference arm: every slot
        vector encoded by the reference's own Encoder (threaded), client
        vectors encrypted with the B200 arm's Rng labels (bit-identical)."""
        from types import SimpleNamespace as NS
        W, d, n, L, spec = self.W, self.d, self.spec.slots, SR.ring.max_level(), self.spec
        client = [[wj] * n for wj in d.w] + [[tk] * n for tk in d.t]
        labels = [400 + j for j in range(8)] + [90, 91, 92]
        for b in blocks:
            client += [d.sugar[b * n:(b + 1) * n], d.bp[b * n:(b + 1) * n]]
            labels += [200 + b, 300 + b]
        t0 = time.perf_counter()
        ms = _timed_encode(SR, client, spec.delta, L, threads)
        t1 = time.perf_counter()
        server = self.server_plaintexts(SR, blocks)
        scale = float(SR.ring.modulus(L))
        pts = _timed_encode(SR, server, scale, L, threads)
        for p in pts:  # eval form for mul_plain (workloads.encode_plaintexts)
            p.ntt_forward()
        t2 = time.perf_counter()
        cts = [SR.ctx.encrypt(SR.sk, m, spec.delta, SR.T.Rng(spec.seed).split(lab), SR.T.Domain.slots)
               for m, lab in zip(ms, labels)]
        q = NS(ct_w=cts[:8], ct_t=cts[8:11])
        nb = len(blocks)
        out = [NS(ct_sugar=cts[11 + 2 * i], ct_bp=cts[12 + 2 * i], pt_attr=pts[8 * i:8 * i + 8], attr_scale=scale,
                  pt_flag=pts[8 * nb + i], flag_scale=scale) for i in range(nb)]
        return (q, out), {"client_vectors": len(client), "client_encode_s": round(t1 - t0, 2),
                          "server_vectors": len(server), "server_encode_s": round(t2 - t1, 2)}

    def ref_step(self, R, SR, chain_r, inp, threads):
        """The reference's own code path: threads over blocks x thresholds
        (protocol.hpp:297-311), per block the ops of workloads.statement_block,
        sum in block order, one inner_sum (protocol.hpp:319-323). Returns
        (count ciphertext, {phase: seconds})."""
        from concurrent.futures import ThreadPoolExecutor
        W, ev, keys = self.W, SR.ev, SR.keys
        q, blocks = inp

        def thr(x, t, norm):
            return R.eval_private_threshold_plain_norm(ev, x, t, norm, chain_r, keys)

        t0 = time.perf_counter()
        with ThreadPoolExecutor(max(1, threads)) as ex:
            risks = list(ex.map(lambda b: W.linear_score(SR, q.ct_w, b.pt_attr, b.attr_scale), blocks))
            futs = [(ex.submit(thr, b.ct_sugar, q.ct_t[0], 1.0), ex.submit(thr, b.ct_bp, q.ct_t[1], 1.0),
                     ex.submit(thr, r, q.ct_t[2], W.RISK_NORM)) for b, r in zip(blocks, risks)]

            def finish(i):
                b, (f1, f2, f3) = blocks[i], futs[i]
                a = ev.rescale(ev.mul_relin(f1.result(), f2.result(), keys))
                a = ev.rescale(ev.mul_relin(a, f3.result(), keys))
                return ev.rescale(ev.mul_plain(a, b.pt_flag, b.flag_scale))

            outs = list(ex.map(finish, range(len(blocks))))
        acc = outs[0]
        for o in outs[1:]:
            acc = ev.add(acc, o)
        t1 = time.perf_counter()
        cnt = R.inner_sum(ev, acc, self.spec.slots, keys)
        return cnt, {"blocks_s": t1 - t0, "slot_sum_s": time.perf_counter() - t1}

    def oracle_check(self, R, W, threads):
        """Blocks 0 and n-1 of the product path as timed (BSGS, record blocks
        as ciphertext batches) vs the BSGS oracle, residue for residue, and
        the decrypted count of their sum + inner_sum in both."""
        import fullsize as F
        # blocks 0 and n-1, plus the block with the most matching records (by
        # the plaintext comparator) so that the sampled count is not trivially 0
        n = self.spec.slots
        d = self.d
        hit = (d.sugar >= d.t[0]) & (d.bp >= d.t[1]) & (d.attrs @ d.w >= d.t[2]) & (d.flag > 0)
        busiest = int(np.argmax(hit[:self.spec.n_cts * n].reshape(self.spec.n_cts, n).sum(axis=1)))
        ids = sorted({0, self.spec.n_cts - 1, busiest})
        SR, chain_r = F.oracle_context(R, W, self.spec, self.S, self.chain)
        outs_r, secs = F.oracle_statement_blocks(R, W, SR, chain_r, self.d, ids, threads)
        keep = []
        self.partial(self.client, 4, self.G.PolyEval.bsgs, keep=keep)
        got = [keep[self.mine.index(b)] for b in ids]
        same = all(F.ct_equal(a, b) for a, b in zip(got, outs_r))
        cnt_g, cnt_r = F.sum_and_count(self.S, got), F.sum_and_count(SR, outs_r)
        return secs, len(ids), {
            "oracle_blocks": ids,
            "bit_exact_vs_oracle_bsgs": bool(same and F.ct_equal(cnt_g, cnt_r)),
            "oracle_decrypted_count": round(F.decrypted_count(SR, cnt_r), 3),
            "gpu_decrypted_count": round(F.decrypted_count(self.S, cnt_g), 3),
            "what": f"blocks {ids} of the product path as timed (BSGS, {self.max_blocks}-block ciphertext batches) "
                    f"vs the BSGS oracle (oracle/bsgs_ref.py over oracle/_ref), residue for residue, and the "
                    f"decrypted count of their sum + inner_sum"}


class LinearScore:
    """Config 2: encrypted linear score per record block, sum_j mul_plain(
    Enc(w_j), pt(attr_j)) + rescale (8 pt x ct MACs); plaintext attributes
    resident on the server, the 8 weight ciphertexts are the query."""
    metric = "encrypted records/sec per linear-score query (8 pt x ct MACs + rescale per block)"
    slot_sum = False
    columns = 1

    def __init__(self, G, W, spec, rank=0, world=1, rotations=True, device=True):
        self.G, self.W, self.spec = G, W, spec
        self.batched, self.max_blocks = True, 8
        self.attrs, self.w = W.linear_score_data(spec)
        if not device:
            return
        from paper_2412_13269_b200 import distributed as D
        self.S = W.make_context(G, spec, relin=False)
        self.chain = None
        self.mine = D.shard(spec.n_cts, world, rank)
        inp = W.config2_inputs(self.S, self.attrs, self.w)
        self.blocks = [inp.blocks[b] for b in self.mine]
        self.plain_scale = inp.plain_scale
        self.client = list(inp.ct_w)

    def partial(self, client, streams, mode, keep=None):
        # one stream: each block is a single plaintext-product-sum launch plus
        # a rescale, too small for host threads to pay off, and the weights'
        # eval form is then computed once per step instead of once per stream
        return [self.W.linear_score(self.S, client, pts, self.plain_scale) for pts in self.blocks]

    def check(self, res):
        n = self.spec.slots
        err = 0.0
        enc = self.G.Encoder(self.S.ring, n)
        for b, ct in zip(self.mine, res):
            got = np.array(enc.decode_slots(self.S.ctx.decrypt(self.S.sk, ct), ct.scale)).real
            want = self.attrs[b * n:(b + 1) * n] @ self.w / self.W.ATTR_NORM
            err = max(err, float(np.max(np.abs(got - want))))
        return {"max_abs_err_vs_plaintext": err, "tolerance": 2.0 ** -20, "within_tolerance": err < 2.0 ** -20}

    def server_plaintexts(self, S, blocks):
        n = self.spec.slots
        return [self.attrs[b * n:(b + 1) * n, j] / self.W.ATTR_NORM for b in blocks for j in range(8)]

    def ref_inputs(self, SR, blocks, threads):
        from types import SimpleNamespace as NS
        n, L, spec = self.spec.slots, SR.ring.max_level(), self.spec
        client = [[wj] * n for wj in self.w]
        t0 = time.perf_counter()
        ms = _timed_encode(SR, client, spec.delta, L, threads)
        t1 = time.perf_counter()
        server = self.server_plaintexts(SR, blocks)
        scale = float(SR.ring.modulus(L))
        pts = _timed_encode(SR, server, scale, L, threads)
        for p in pts:
            p.ntt_forward()
        t2 = time.perf_counter()
        ct_w = [SR.ctx.encrypt(SR.sk, m, spec.delta, SR.T.Rng(spec.seed).split(400 + j), SR.T.Domain.slots)
                for j, m in enumerate(ms)]
        out = [NS(pts=pts[8 * i:8 * i + 8], scale=scale) for i in range(len(blocks))]
        return (ct_w, out), {"client_vectors": len(client), "client_encode_s": round(t1 - t0, 2),
                             "server_vectors": len(server), "server_encode_s": round(t2 - t1, 2)}

    def ref_step(self, R, SR, chain_r, inp, threads):
        from concurrent.futures import ThreadPoolExecutor
        ct_w, blocks = inp
        t0 = time.perf_counter()
        with ThreadPoolExecutor(max(1, threads)) as ex:  # one block per thread (protocol.hpp:297-311)
            out = list(ex.map(lambda b: self.W.linear_score(SR, ct_w, b.pts, b.scale), blocks))
        return out, {"blocks_s": time.perf_counter() - t0, "slot_sum_s": 0.0}

    def oracle_check(self, R, W, threads):
        """Every block's score through the reference's own mul_plain/add/
        rescale vs the product's, residue for residue."""
        import fullsize as F
        SR, _ = F.oracle_context(R, W, self.spec, self.S, None, rotations=False)
        inp = W.config2_inputs(SR, self.attrs, self.w)
        t0 = time.perf_counter()
        ref = [W.linear_score(SR, inp.ct_w, inp.blocks[b], inp.plain_scale) for b in self.mine]
        secs = time.perf_counter() - t0
        got = self.partial(self.client, 1, None)
        return secs, len(ref), {"oracle_blocks": list(self.mine),
                                "bit_exact_vs_reference": all(F.ct_equal(a, b) for a, b in zip(got, ref)),
                                "what": "every block's score vs the reference's mul_plain/add/rescale"}


WORKLOADS = {2: LinearScore, 3: ThresholdCount, 4: Statement, 5: Statement}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def run_b200(args):
    import torch

    from paper_2412_13269_b200 import tetris as G
    from paper_2412_13269_b200 import workloads as W

    world, rank, local = dist_env()
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    if G.device_count() < 1:
        raise SystemExit("bench.py: no CUDA device visible (the B200 arm has no CPU fallback)")
    G.set_default_device(local)

    spec = W.CONFIGS[args.config]
    if args.K or args.group:  # gadget / special-prime experiments
        import dataclasses
        spec = dataclasses.replace(spec, K=args.K or spec.K, group=args.group or spec.group)
    t0 = time.time()
    from paper_2412_13269_b200 import distributed as D
    wl = WORKLOADS[args.config](G, W, spec, rank, world, rotations=(rank == 0))
    wl.batched, wl.max_blocks = not args.no_batch, args.max_blocks
    S, chain = wl.S, wl.chain
    D.check_exact(world, S.primes)
    S.ring.synchronize()
    log(f"[rank {rank}] setup {time.time() - t0:.1f}s: {spec.name} N={spec.N} L={spec.nq - 1} K={spec.K} "
        f"blocks={wl.mine}")
    # stream-ordered pool grown once up front: no memory mapping inside timed steps
    G.pool_reserve(S.ring, int(args.pool_gb * (1 << 30)))
    mode = G.PolyEval.bsgs if args.poly_eval == "bsgs" else G.PolyEval.ladder
    ext = torch.cuda.ExternalStream(S.ring.stream_handle(), device=torch.device("cuda", local))
    flush = torch.empty(64 << 22, dtype=torch.int32, device="cuda")  # 1 GiB > 126 MB L2
    out_meta = {}

    def query(client, streams=None, ready=None):
        streams = streams or args.streams
        # record blocks run concurrently (one host thread + CUDA stream each);
        # outputs are summed in block order
        acc = wl.partial(client, streams, mode, ready=ready) if ready else wl.partial(client, streams, mode)
        if not wl.slot_sum:  # per-block results stay on their rank (no exchange)
            return acc
        if world > 1:
            if "level" not in out_meta:  # ranks without blocks learn the output level once
                lv = torch.tensor([acc.level() if acc is not None else -1], device="cuda", dtype=torch.int64)
                dist.all_reduce(lv, op=dist.ReduceOp.MAX)
                out_meta["level"] = int(lv.item())
            if acc is None:  # contributes zero
                acc = S.ctx.zero_ciphertext(out_meta["level"], 1.0, S.sk.id(), G.Domain.slots)
            reduce_partial_to_root(G, torch, dist, acc, ext, spec.N)
        if rank == 0:
            acc = G.inner_sum(S.ev, acc, spec.slots, S.keys)
        return acc

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        S.ring.synchronize()

    def timed(fn, steps):
        times = []
        out = None
        for _ in range(steps):
            with torch.cuda.stream(ext):
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(ext)
            out = fn()
            b.record(ext)
            times.append((a, b))
        S.ring.synchronize()
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in times], out

    def fresh_query(streams=None):
        # every step pays the whole query: memoised eval forms of the client
        # ciphertexts (weights' forward NTTs) from the previous step dropped
        for c in wl.client:
            c.clear_eval_cache()
        return query(wl.client, streams)

    # warm-up
    for _ in range(args.warmup):
        res = fresh_query()
    barrier()
    # timed region (device-resident inputs)
    prof_region = os.environ.get("TG_PROFILE_REGION") == "1"  # ncu --profile-from-start off
    try:  # NVML handle by PCI address (CUDA and NVML indices can differ)
        pr = torch.cuda.get_device_properties(local)
        pci = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
    except Exception:
        pci = None
    with ClockSampler(local, pci) as clocks:
        barrier()
        if prof_region:
            torch.cuda.cudart().cudaProfilerStart()
        ms_list, res = timed(fresh_query, args.steps)
        if prof_region:
            torch.cuda.cudart().cudaProfilerStop()
        barrier()
    ms_step = sum(ms_list) / len(ms_list)
    log(f"[rank {rank}] step ms: " + " ".join(f"{m:.1f}" for m in ms_list))
    if world > 1:
        tt = torch.tensor([ms_step], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_step = float(tt.item())
    records = spec.records
    value = records / (ms_step / 1e3)

    # the same query on ONE stream, unprofiled: with the profiled replay's
    # kernel sum below this gives the GPU idle per step of serial issue
    barrier()
    single_list, _ = timed(lambda: fresh_query(streams=1), args.steps)
    single_ms = sum(single_list) / len(single_list)

    # profiled replay of the same steps: per-kernel-class CUDA-event times
    G.profile_enable(S.ring, True)
    barrier()
    # one stream here, so every kernel's event-bracketed duration is its own
    # (concurrent streams would time-share the SMs inside the brackets)
    _, _ = timed(lambda: fresh_query(streams=1), args.steps)
    prof = G.profile_read(S.ring)
    G.profile_enable(S.ring, False)

    # end to end through the public API: the query's client ciphertexts come
    # from pinned host memory every step, the count goes back to the host
    # all client ciphertexts in one pinned buffer -> one H2D DMA per step
    metas, off = [], 0
    for c in wl.client:
        metas.append((off, len(c.parts), c.level(), c.scale, c.sk_id))
        off += len(c.parts) * (c.level() + 1) * spec.N
    host_buf = G.pinned_empty([off])
    for c, m in zip(wl.client, metas):
        n = m[1] * (m[2] + 1) * spec.N
        G.ciphertext_to_numpy(c, host_buf[m[0]:m[0] + n])
    res_list = res if isinstance(res, list) else [res]
    host_out = [G.pinned_empty([len(c.parts), c.level() + 1, spec.N]) for c in res_list] \
        if (rank == 0 or not wl.slot_sum) else []

    uploader = G.HostUpload(S.ring, host_buf, metas, G.Form.coeff, G.Domain.slots)

    groups = getattr(wl, "upload_groups", None) if not args.no_staged_upload else None

    def e2e_step():
        if groups:  # every step: pinned host -> HBM, one DMA per input group on a copy
            # stream; each job waits (on the device) for its own group only
            ups = uploader.upload_async([hi - lo for lo, hi in groups.values()])
            r = query(ups, ready=lambda name: uploader.wait(list(range(*groups[name]))))
        else:  # every step: pinned host -> HBM, one DMA
            r = query(uploader.upload())
        if host_out:  # the result back on the host every step
            for c, h in zip(r if isinstance(r, list) else [r], host_out):
                G.ciphertext_to_numpy(c, h)
        return r

    for _ in range(max(2, args.warmup)):
        e2e_step()
    barrier()
    e2e_ms_list, _ = timed(e2e_step, args.steps)
    e2e_ms = sum(e2e_ms_list) / len(e2e_ms_list)
    log(f"[rank {rank}] e2e step ms: " + " ".join(f"{m:.1f}" for m in e2e_ms_list))
    res_b, used_hi = G.pool_stats(S.ring)
    log(f"[rank {rank}] pool reserved {res_b / 2**30:.1f} GiB, used high-water {used_hi / 2**30:.1f} GiB")
    if world > 1:
        tt = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    h2d = int(host_buf.nbytes)
    d2h = int(sum(h.nbytes for h in host_out))

    # decrypt + check the count (rank 0)
    check = {}
    if rank == 0:
        check = wl.check(res)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # roofline: dominant kernel class by device time
    peak, peak_kind = measured_peaks()
    dom = max(prof.items(), key=lambda kv: kv[1][0])
    dname, (dms, dn, dbytes) = dom[0], dom[1][:3]
    per_launch_ms = dms / dn
    achieved = (dbytes / dn) / (per_launch_ms / 1e3) / 1e9
    total_prof_ms = sum(v[0] for v in prof.values())
    launches = sum(v[1] for v in prof.values()) // args.steps * args.steps  # kernel launches (tg_profile_read)
    # DRAM traffic per launch of the dominant class from the committed ncu
    # capture of this workload (profiles/traffic_<workload>.json), else null
    traffic = None
    tf = ROOT / "profiles" / f"traffic_{spec.name}.json"
    if tf.exists():
        tcls = json.loads(tf.read_text()).get("classes", {}).get(dname)
        if tcls:
            traffic = {"bytes_per_launch": tcls["dram_bytes_per_launch"],
                       "vs_algorithmic": round(tcls["dram_bytes_per_launch"] / (dbytes / dn), 3),
                       "source": str(tf.relative_to(ROOT))}
    roofline = {"bound": "hbm", "kernel": dname, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4),
                # DRAM bytes per launch of the dominant class (ncu capture), details alongside
                "traffic": round(traffic["bytes_per_launch"]) if traffic else None, "traffic_detail": traffic,
                "peak_kind": peak_kind,
                "bytes_per_launch": dbytes / dn, "ms_per_launch": per_launch_ms,
                "share_of_step": round(dms / total_prof_ms, 3),
                # the NTT's actual bound is the FP64 pipe: algorithmic
                # FP64 ops = 8 per butterfly (exact modmul 6 + add/sub 2), N/2 log N
                # butterflies per row = bytes * log N / 4, against the measured pipe peak
                "fp64": fp64_roofline(prof, spec.N) if dname.startswith("ntt") else fp64_roofline_class(prof, dname),
                "per_kernel": {k: {"ms": round(v[0] / args.steps, 4), "launches": v[1] // args.steps,
                                   "GBps": round((v[2] / v[1]) / ((v[0] / v[1]) / 1e3) / 1e9, 1)}
                               for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}}

    # server-side plaintext encoding (reported as its own line,
    # outside the query): this shard's slot vectors -> plaintexts on the device
    server_enc = None
    if hasattr(wl, "server_plaintexts"):
        vecs = wl.server_plaintexts(S, wl.mine)
        with torch.cuda.stream(ext):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            W.encode_plaintexts(S, vecs, S.ring.max_level())  # warm
            S.ring.synchronize()
            a.record(ext)
            W.encode_plaintexts(S, vecs, S.ring.max_level())
            b.record(ext)
        S.ring.synchronize()
        ms = a.elapsed_time(b)
        server_enc = {"vectors": len(vecs), "ms": round(ms, 3),
                      "records_per_s": round(len(wl.mine) * spec.slots / (ms / 1e3), 1),
                      "what": "Encoder::encode_slots at scale q_L + forward NTT of the shard's server plaintexts "
                              "(tg_encode_slots, one launch), device-timed; not inside the query (the reference's "
                              "p-dependent accounting, cli.hpp:240-244)"}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(G, W, spec, wl)
        except Exception as e:  # the baseline is reported, never the product
            cpu = {"value": None, "error": str(e)[:300]}

    clk = clocks.summary()
    line = {
        "metric": wl.metric,
        "value": round(value, 1), "unit": "records/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64 (mod-q RNS residues)", "data": "synthetic",
        "config": workload_config(spec),
        "amortized_us_per_record": round(ms_step * 1e3 / records, 4),
        "impl_detail": {"poly_eval": args.poly_eval, "streams": args.streams,
                        "batched": bool(getattr(wl, "batched", False)),
                        "max_blocks": getattr(wl, "max_blocks", None), "parallelism": f"block-shard x{world}",
                        "l2": "1 GiB buffer written between timed steps; working set (keys, blocks) > 126 MB L2",
                        "inputs": "client ciphertexts device-resident; their memoised eval forms dropped every step"},
        "check": check,
        "e2e": {"value": round(records / (e2e_ms / 1e3), 1), "unit": "records/s", "ms_per_step": round(e2e_ms, 3),
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches // args.steps),
        "gpu_time": {"kernel_sum_ms": round(total_prof_ms / args.steps, 3),
                     "single_stream_ms": round(single_ms, 3), "concurrent_ms": round(ms_step, 3),
                     "single_stream_idle_ms": round(single_ms - total_prof_ms / args.steps, 3),
                     "note": "kernel_sum: per-op CUDA-event brackets on one stream (profiled replay); single_stream: "
                             "the same query on one stream, unprofiled; concurrent: the timed step (--streams "
                             "pipelines) - below kernel_sum where pipelines overlap"},
        "roofline": roofline,
        "server_encode": server_enc,
        "cpu_baseline": cpu,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def workload_config(spec):
    """The workload (BASELINE.json config) both arms run: identical dicts, so
    the driver's same-config check compares like with like. Implementation
    choices (evaluator, batching, threads) go in impl_detail."""
    cfg = {"workload": spec.name, "records": spec.records, "N": spec.N, "levels": spec.nq - 1,
           "q_bits": spec.q_bits, "special_primes": f"{spec.K}x{spec.sp_bits}b", "dnum": -(-spec.nq // spec.group),
           "record_blocks": spec.n_cts, "slots": spec.slots, "secret_hw": spec.h, "seed": spec.seed}
    if spec.degrees:
        cfg.update({"chain_degrees": list(spec.degrees), "alpha": spec.alpha, "epsilon": spec.epsilon})
    return cfg


def host_cpu():
    model = "unknown"
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count() or 1, "model": model}


# ---------------------------------------------------------------------------
# CPU reference: the compiled, unmodified reference (oracle/_ref)
# ---------------------------------------------------------------------------
def _ref_module():
    sys.path.insert(0, str(ROOT / "tests"))
    from common import load_ref
    return load_ref()


def load_workloads():
    """paper_2412_13269_b200/workloads.py by path (numpy only): the reference
    arm must not import the package, whose __init__ loads the B200 library."""
    import importlib.util
    if "paper_2412_13269_b200.workloads" in sys.modules:
        return sys.modules["paper_2412_13269_b200.workloads"]
    name = "tg_workloads_standalone"
    if name not in sys.modules:
        sp = importlib.util.spec_from_file_location(name, ROOT / "paper_2412_13269_b200" / "workloads.py")
        mod = importlib.util.module_from_spec(sp)
        sys.modules[name] = mod
        sp.loader.exec_module(mod)
    return sys.modules[name]


def cpu_baseline(G, W, spec, wl):
    """Bounded sample (~10-60 s of CPU work) of the same workload through the
    oracle on the host cores, compared residue for residue with the product
    path exactly as timed (wl.oracle_check): configs 4/5 blocks 0 and n-1
    through the BSGS oracle (oracle/bsgs_ref.py over oracle/_ref), plus the
    decrypted count of their sum + inner_sum in both; config 3 the whole
    query; config 2 every block through the reference's own ops."""
    R = _ref_module()
    if R is None:
        raise RuntimeError("oracle/_ref not built")
    nblk = min(spec.n_cts, 3) if isinstance(wl, Statement) else spec.n_cts
    threads = max(1, min(nblk * wl.columns, os.cpu_count() or 1))
    secs, nb, chk = wl.oracle_check(R, W, threads)
    recs = nb * spec.slots
    kind = "port" if spec.degrees else "reference"
    return {"value": round(recs / secs, 2), "unit": "records/s", "cores": threads, "kind": kind,
            "sample": f"{nb} record block(s) x {spec.slots} records through "
                      + ("the BSGS oracle (oracle/bsgs_ref.py: the product's BSGS order restated over the compiled "
                         "reference's Evaluator primitives, oracle/_ref, g++ -O2)" if spec.degrees else
                         "the reference's own ops (oracle/_ref, g++ -O2)")
                      + f" on {threads} thread(s), {secs:.2f} s"
                      + ("; config 3 includes the inner_sum" if isinstance(wl, ThresholdCount) else ""),
            "seconds": round(secs, 2), **chk, "host": host_cpu()}


def ref_threads(wl, nblocks):
    """Host threads the reference uses: one per threshold job (protocol.hpp:297-311)."""
    return max(1, min(nblocks * wl.columns, os.cpu_count() or 1))


def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    headers, g++ -O2) on this host's cores, on the same workload config as the
    B200 arm. Nothing from paper_2412_13269_b200 is imported or loaded here:
    inputs are encoded by the reference's Encoder (threaded over vectors) and
    encrypted with the same seeds as the B200 arm's."""
    world, rank, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    W = load_workloads()
    spec = W.CONFIGS[args.config]
    R = _ref_module()
    if R is None:
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref not built (needs /root/reference at build time)"}))
        return
    cores = os.cpu_count() or 1
    cls = WORKLOADS[args.config]
    nblk = spec.n_cts if cls is LinearScore else max(1, min(spec.n_cts, cores // cls.columns))
    blocks = list(range(nblk))
    t0 = time.time()
    wl = cls(None, W, spec, device=False)
    SR = W.make_context(R, spec, rotations=W.inner_sum_rotations(spec.slots) if wl.slot_sum else [],
                        relin=bool(spec.degrees))
    chain = W.config3_chain(R, spec) if spec.degrees else None
    threads = ref_threads(wl, nblk)
    inp, enc = wl.ref_inputs(SR, blocks, cores)
    log(f"[reference] setup {time.time() - t0:.1f}s, sample {nblk} blocks on {threads} threads, encode {enc}")

    # one record block on ONE thread, once (the reference's single-threaded figure)
    one = None
    if not args.no_1thread and nblk >= 1:
        sub = (inp[0][:1], inp[1]) if cls is ThresholdCount else (inp[0], inp[1][:1])
        _, ph = wl.ref_step(R, SR, chain, sub, 1)
        s1 = ph["blocks_s"] + ph["slot_sum_s"]
        one = {"value": round(spec.slots / s1, 2), "unit": "records/s", "cores": 1, "seconds": round(s1, 2),
               "sample": "record block 0 through the same code path on one thread" +
                         (", incl. the slot-sum of its output" if wl.slot_sum else "")}

    phases = []

    def step():
        t = time.perf_counter()
        _, ph = wl.ref_step(R, SR, chain, inp, threads)
        phases.append(ph)
        return time.perf_counter() - t

    for _ in range(args.warmup):
        step()
    phases.clear()
    secs = [step() for _ in range(args.steps)]
    s = sum(secs) / len(secs)
    recs = nblk * spec.slots
    value = recs / s
    blk_s = sum(p["blocks_s"] for p in phases) / len(phases)
    ss_s = sum(p["slot_sum_s"] for p in phases) / len(phases)
    sample = (f"each step = {nblk} of {spec.n_cts} record blocks ({recs} records) through the reference's own code "
              f"path on {threads} threads (unmodified headers, g++ -O2; the reference's T_k-ladder polynomial "
              f"evaluator)" + (", then the sum and ONE inner_sum of the sample's output inside the step "
                               f"({ss_s:.2f} s of {s:.2f} s)" if wl.slot_sum else "")
              + "; per-record work is identical across blocks")
    # server plaintext encoding by the reference's own encoder, as its own line
    senc = None
    if enc.get("server_vectors"):
        senc = {"vectors": enc["server_vectors"], "seconds": enc["server_encode_s"], "threads": cores,
                "records_per_s": round(nblk * spec.slots / enc["server_encode_s"], 2),
                "what": "Encoder::encode_slots (O(n^2) DFT, ckks.hpp:59-86) at scale q_L + NTT of the sample's "
                        "server plaintexts, vectors spread over a std::thread pool; not inside the query"}
    print(json.dumps({
        "impl": "reference", "metric": cls.metric,
        "value": round(value, 2), "unit": "records/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(s * 1e3, 1), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64 (mod-q RNS residues)", "data": "synthetic",
        "config": workload_config(spec),
        "amortized_us_per_record": round(s * 1e6 / recs, 2),
        "impl_detail": {"poly_eval": "ladder (reference eval_chebyshev)", "threads": threads,
                        "sample_records": recs, "blocks_s": round(blk_s, 3), "slot_sum_s": round(ss_s, 3)},
        "cpu_baseline": {"value": round(value, 2), "unit": "records/s", "cores": threads, "kind": "reference",
                         "sample": sample, "host": host_cpu()},
        "cpu_1thread": one,
        "server_encode": senc,
        "e2e": {"value": round(value, 2), "unit": "records/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "product_loaded": any(m.startswith("paper_2412_13269_b200") for m in sys.modules),
    }), flush=True)


# ---------------------------------------------------------------------------
# Config 1 (BASELINE.json configs[0]): the CKKS ring-op microbench
# ---------------------------------------------------------------------------
CONFIG1_METRIC = ("ciphertexts/sec through the config-1 ring-op sequence (forward NTT, inverse NTT, tensor + "
                  "relinearisation with ct_(i+1 mod 64), rescale, rotation by 1; every op on all 64 ciphertexts)")


def config1_inputs(T, W, spec, n_cts):
    """64 ciphertexts of uniform residues (sample_uniform per part from
    Rng(seed).split(5).split(2i + j)), keys from the workload's keygen."""
    S = W.make_context(T, spec, rotations=(1,))
    rng = T.Rng(spec.seed).split(5)
    L = S.ring.max_level()
    cts = []
    for i in range(n_cts):
        c = T.Ciphertext()
        c.parts = [T.sample_uniform(S.ring, L, 0, rng.split(2 * i + j)) for j in range(2)]
        c.scale, c.domain, c.sk_id = spec.delta, T.Domain.slots, S.sk.id()
        cts.append(c)
    return S, cts


def config1_ops(ev, keys, x, y, x_eval):
    """One step: every op of the config on the whole batch. Inputs are fresh
    exclusively owned blocks (mul by 1 costs one HBM pass, counted as
    scalar_copy) so the transforms are real, not memoised; the shared inputs'
    memoised eval forms are dropped first, so the product pays its operands'
    forward transforms every step."""
    x.clear_eval_cache()
    y.clear_eval_cache()
    f = ev.mul_scalar(x, 1.0, 1.0)
    f.to_eval()                                   # forward NTT, 64 x 2 x 8 rows
    g = ev.mul_scalar(x_eval, 1.0, 1.0)
    g.to_coeff()                                  # inverse NTT
    pr = ev.rescale(ev.mul_relin(x, y, keys))     # tensor + relinearisation, rescale
    rot = ev.rotate(x, 1, keys)                   # rotation by 1 (5^1)
    return f, g, pr, rot


def run_config1(args):
    import torch

    from paper_2412_13269_b200 import tetris as G
    from paper_2412_13269_b200 import workloads as W

    world, rank, local = dist_env()
    if world > 1:  # every rank runs its own 64 ciphertexts (weak scaling, no exchange)
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist = None
        torch.cuda.set_device(local)
    if G.device_count() < 1:
        raise SystemExit("bench.py: no CUDA device visible (the B200 arm has no CPU fallback)")
    G.set_default_device(local)
    spec = W.CONFIGS[1]
    n = spec.n_cts
    S, cts = config1_inputs(G, W, spec, n)
    ev, keys, ring = S.ev, S.keys, S.ring
    x = G.stack_ciphertexts(cts)
    y = G.stack_ciphertexts(cts[1:] + cts[:1])
    x_eval = x.copy()
    x_eval.to_eval()
    G.pool_reserve(ring, int(min(args.pool_gb, 16.0) * (1 << 30)))  # no pool growth inside timed steps
    ext = torch.cuda.ExternalStream(ring.stream_handle(), device=torch.device("cuda", local))
    flush = torch.empty(64 << 22, dtype=torch.int32, device="cuda")

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        ring.synchronize()

    def timed(fn, steps):
        ev_pairs = []
        out = None
        for _ in range(steps):
            with torch.cuda.stream(ext):
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(ext)
            out = fn()
            b.record(ext)
            ev_pairs.append((a, b))
        ring.synchronize()
        torch.cuda.synchronize()
        return [a.elapsed_time(b) for a, b in ev_pairs], out

    step = lambda: config1_ops(ev, keys, x, y, x_eval)  # noqa: E731
    for _ in range(args.warmup):
        step()
    barrier()
    try:
        pr_ = torch.cuda.get_device_properties(local)
        pci = f"{pr_.pci_domain_id:08x}:{pr_.pci_bus_id:02x}:{pr_.pci_device_id:02x}.0"
    except Exception:
        pci = None
    with ClockSampler(local, pci) as clocks:
        barrier()
        ms_list, outs = timed(step, args.steps)
        barrier()
    ms = sum(ms_list) / len(ms_list)
    log(f"[rank {rank}] config-1 step ms: " + " ".join(f"{m:.3f}" for m in ms_list))
    if dist is not None:
        tt = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    # per-op device times (one op per timed bracket) and kernel classes
    per_op = {}
    for name, fn in (("scalar_copy", lambda: ev.mul_scalar(x, 1.0, 1.0)),
                     ("ntt_fwd", lambda: config1_ops(ev, keys, x, y, x_eval)[0]),
                     ("tensor_relin_rescale", lambda: (x.clear_eval_cache(), y.clear_eval_cache(),
                                                       ev.rescale(ev.mul_relin(x, y, keys)))[-1]),
                     ("rotate_1", lambda: ev.rotate(x, 1, keys))):
        if name == "ntt_fwd":
            def fn():  # noqa: F811
                f = ev.mul_scalar(x, 1.0, 1.0)
                f.to_eval()
                return f
        t, _ = timed(fn, max(3, args.steps))
        per_op[name] = round(sum(t) / len(t), 4)
    G.profile_enable(ring, True)
    barrier()
    timed(step, args.steps)
    prof = G.profile_read(ring)
    G.profile_enable(ring, False)

    # end to end: the 64 ciphertexts from pinned host memory every step, the
    # relinearised-rescaled products and the rotations back to the host
    limbs = spec.nq
    host_in = G.pinned_empty([n * 2 * limbs * spec.N])
    metas = []
    for i, c in enumerate(cts):
        off = i * 2 * limbs * spec.N
        metas.append((off, 2, c.level(), c.scale, c.sk_id))
        G.ciphertext_to_numpy(c, host_in[off:off + 2 * limbs * spec.N])
    up = G.HostUpload(ring, host_in, metas, G.Form.coeff, G.Domain.slots)
    host_pr = G.pinned_empty([2 * n, limbs - 1, spec.N])
    host_rot = G.pinned_empty([2 * n, limbs, spec.N])

    def e2e_step():
        c = up.upload()
        xx = G.stack_ciphertexts(c)
        yy = G.stack_ciphertexts(c[1:] + c[:1])
        xe = xx.copy()
        xe.to_eval()
        o = config1_ops(ev, keys, xx, yy, xe)
        G.ciphertext_to_numpy(o[2], host_pr)
        G.ciphertext_to_numpy(o[3], host_rot)
        return o

    for _ in range(max(2, args.warmup)):
        e2e_step()
    barrier()
    e2e_list, _ = timed(e2e_step, args.steps)
    e2e_ms = sum(e2e_list) / len(e2e_list)
    if dist is not None:
        tt = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
        if rank != 0:
            dist.destroy_process_group()
            return

    peak, peak_kind = measured_peaks()
    dname, (dms, dn, dbytes) = (lambda kv: (kv[0], kv[1][:3]))(max(prof.items(), key=lambda kv: kv[1][0]))
    per_launch = dms / dn
    achieved = (dbytes / dn) / (per_launch / 1e3) / 1e9
    total = sum(v[0] for v in prof.values())
    mib = 1 << 20
    limb = spec.N * 8
    # SURVEY 8(d) config-1 totals (algorithmic bytes; limb-poly = N*8 B)
    alg = {"ntt_fwd": 2 * n * 2 * limbs * limb, "ntt_inv": 2 * n * 2 * limbs * limb,
           "tensor_relin_rescale": (6 * limbs + (4 * limbs - 2)) * n * limb
           + 2 * (-(-limbs // spec.group)) * (limbs + spec.K) * limb,
           "rotate_1": (4 * limbs) * n * limb + 2 * (-(-limbs // spec.group)) * (limbs + spec.K) * limb}
    net_fwd = per_op["ntt_fwd"] - per_op["scalar_copy"]
    ops = {"ntt_fwd": {"ms": round(net_fwd, 4), "GBps": round(alg["ntt_fwd"] / (net_fwd / 1e3) / 1e9, 1),
                       "note": "net of the exclusive copy"},
           "tensor_relin_rescale": {"ms": per_op["tensor_relin_rescale"],
                                    "GBps": round(alg["tensor_relin_rescale"] / (per_op["tensor_relin_rescale"] / 1e3)
                                                  / 1e9, 1)},
           "rotate_1": {"ms": per_op["rotate_1"],
                        "GBps": round(alg["rotate_1"] / (per_op["rotate_1"] / 1e3) / 1e9, 1)}}
    for k in ops:
        ops[k]["frac_of_hbm"] = round(ops[k]["GBps"] / peak, 4)
        ops[k]["alg_MiB"] = round(alg[k] / mib, 1)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = config1_cpu_baseline(G, W, spec, outs)
        except Exception as e:
            cpu = {"value": None, "error": str(e)[:300]}
    line = {
        "metric": CONFIG1_METRIC, "value": round(world * n / (ms / 1e3), 1), "unit": "ciphertexts/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64 (mod-q RNS residues)",
        "data": "synthetic", "config": workload_config(spec),
        "impl_detail": {"batch": n, "parallelism": f"replicas x{world} (no exchange)",
                        "l2": "1 GiB buffer written between timed steps"},
        "per_op": ops,
        "e2e": {"value": round(world * n / (e2e_ms / 1e3), 1), "unit": "ciphertexts/s", "ms_per_step": round(e2e_ms, 4),
                "h2d_bytes_per_step": int(host_in.nbytes), "d2h_bytes_per_step": int(host_pr.nbytes + host_rot.nbytes)},
        "gpu_launches": int(sum(v[1] for v in prof.values()) // args.steps),
        "roofline": {"bound": "hbm", "kernel": dname, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None, "peak_kind": peak_kind,
                     "bytes_per_launch": dbytes / dn, "ms_per_launch": per_launch,
                     "share_of_step": round(dms / total, 3),
                     "per_kernel": {k: {"ms": round(v[0] / args.steps, 4), "launches": v[1] // args.steps,
                                        "GBps": round((v[2] / v[1]) / ((v[0] / v[1]) / 1e3) / 1e9, 1)}
                                    for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}},
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def config1_cpu_baseline(G, W, spec, outs):
    """The reference (oracle/_ref) on a 4-ciphertext sample, one thread: the
    same ops, compared residue for residue with the device batch."""
    R = _ref_module()
    if R is None:
        raise RuntimeError("oracle/_ref not built")
    k = 4
    SR, rc = config1_inputs(R, W, spec, k)
    t0 = time.perf_counter()
    ref = config1_ref_ops(SR, rc)
    secs = time.perf_counter() - t0
    got_pr = G.unstack_ciphertext(outs[2])
    got_rot = G.unstack_ciphertext(outs[3])
    same = all(np.array_equal(a.to_numpy(), b.to_numpy())
               for i in range(k - 1) for a, b in zip(got_pr[i].parts, ref["pr"][i].parts))
    same &= all(np.array_equal(a.to_numpy(), b.to_numpy())
                for i in range(k) for a, b in zip(got_rot[i].parts, ref["rot"][i].parts))
    return {"value": round(k / secs, 3), "unit": "ciphertexts/s", "cores": 1, "kind": "reference",
            "sample": f"{k} ciphertexts through the reference's own ops (forward + inverse NTT of both parts, "
                      f"mul_relin + rescale, rotate by 1; unmodified headers, g++ -O2) on one thread, {secs:.2f} s",
            "seconds": round(secs, 2), "bit_exact_vs_reference_sample": bool(same), "host": host_cpu()}


def config1_ref_ops(SR, rc):
    ev, keys = SR.ev, SR.keys
    k = len(rc)
    for c in rc:
        for p in c.parts:
            e = SR.T.ntt_transform(p, SR.T.Form.eval)
            SR.T.ntt_transform(e, SR.T.Form.coeff)
    pr = [ev.rescale(ev.mul_relin(rc[i], rc[(i + 1) % k], keys)) for i in range(k - 1)]
    rot = [ev.rotate(c, 1, keys) for c in rc]
    return {"pr": pr, "rot": rot}


def run_config1_reference(args):
    """Reference arm, config 1: the reference's own ops on every host core
    (one ciphertext per thread), a sample of cores ciphertexts per step."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    W = load_workloads()
    spec = W.CONFIGS[1]
    R = _ref_module()
    if R is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    from concurrent.futures import ThreadPoolExecutor
    cores = os.cpu_count() or 1
    k = max(2, min(spec.n_cts, cores))
    SR, rc = config1_inputs(R, W, spec, k)
    ev, keys = SR.ev, SR.keys

    def one(i):
        c = rc[i]
        for p in c.parts:
            SR.T.ntt_transform(SR.T.ntt_transform(p, SR.T.Form.eval), SR.T.Form.coeff)
        ev.rescale(ev.mul_relin(c, rc[(i + 1) % k], keys))
        ev.rotate(c, 1, keys)

    def step():
        t = time.perf_counter()
        with ThreadPoolExecutor(k) as ex:
            list(ex.map(one, range(k)))
        return time.perf_counter() - t

    for _ in range(args.warmup):
        step()
    secs = [step() for _ in range(args.steps)]
    s = sum(secs) / len(secs)
    value = k / s
    print(json.dumps({
        "impl": "reference", "metric": CONFIG1_METRIC, "value": round(value, 3), "unit": "ciphertexts/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(s * 1e3, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64 (mod-q RNS residues)",
        "data": "synthetic", "config": workload_config(spec),
        "cpu_baseline": {"value": round(value, 3), "unit": "ciphertexts/s", "cores": k, "kind": "reference",
                         "sample": f"each step = {k} of {spec.n_cts} ciphertexts, one per thread, through the "
                                   f"reference's own ops (NTT fwd+inv of both parts, mul_relin + rescale, rotate by 1; "
                                   f"unmodified headers, g++ -O2)", "host": host_cpu()},
        "e2e": {"value": round(value, 3), "unit": "ciphertexts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "product_loaded": any(m.startswith("paper_2412_13269_b200") for m in sys.modules),
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=4, help="concurrent pipelines (host thread + CUDA stream each) per GPU")
    ap.add_argument("--poly-eval", choices=["bsgs", "ladder"], default="bsgs",
                    help="Chebyshev evaluator of the sign stages (BASELINE configs specify BSGS)")
    ap.add_argument("--no-staged-upload", action="store_true",
                    help="e2e: one synchronous upload per step instead of per-group DMAs overlapping compute")
    ap.add_argument("--no-batch", action="store_true",
                    help="statement workloads: one ciphertext per pipeline instead of ciphertext batches")
    ap.add_argument("--max-blocks", type=int, default=8, help="record blocks per ciphertext batch")
    ap.add_argument("--pool-gb", type=float, default=48.0, help="device memory pool reserved up front (GiB)")
    ap.add_argument("--K", type=int, default=0, help="override the special-prime count (experiments)")
    ap.add_argument("--group", type=int, default=0, help="override the gadget group size (experiments)")
    ap.add_argument("--no-1thread", action="store_true", help="reference arm: skip the one-thread row")
    ap.add_argument("--config", type=int, choices=[1, 2, 3, 4, 5], default=4,
                    help="BASELINE.json workload: 4 = full TETRIS statement (default), 3 = threshold count, "
                         "5 = scale-out stress, 2 = linear score, 1 = ring-op microbench")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.config == 1:
        (run_config1_reference if args.impl == "reference" else run_config1)(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
