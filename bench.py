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


class ThresholdCount:
    """Config 3: private threshold of every encrypted score block against an
    encrypted threshold (plain norm), summed."""
    metric = "encrypted records/sec per TETRIS threshold-count query (amortized us/record in config)"
    slot_sum = True

    def check(self, res):
        return decrypted_count(self.G, self.S, self.spec, res, self.plain_count())

    def __init__(self, G, W, spec, rank=0, world=1, rotations=True, device=True):
        from paper_2412_13269_b200 import distributed as D
        self.G, self.W, self.spec = G, W, spec
        self.batched, self.max_blocks = True, 8
        self.scores, self.thr, _, _ = W.linear_scores(spec)
        if not device:  # inputs only (the CPU reference arm)
            return
        rot = W.inner_sum_rotations(spec.slots) if rotations else []
        self.S = W.make_context(G, spec, rotations=rot)
        self.chain = W.config3_chain(G, spec)
        self.mine = D.shard(spec.n_cts, world, rank)
        cts, ct_t, _, _ = W.config3_inputs(self.S, ct_indices=self.mine, scores=self.scores, t=self.thr)
        self.client = cts + [ct_t]

    def partial(self, client, streams, mode):
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
        acc = outs[0]
        for o in outs[1:]:
            acc = self.S.ev.add(acc, o)
        return acc

    def plain_count(self):
        return int((self.scores >= self.thr).sum())

    def ref_inputs(self, R, SR, chain_r, host_encode, blocks):
        n = self.spec.slots
        cts = [host_encode(self.scores[b * n:(b + 1) * n], 100 + b) for b in blocks]
        return cts, host_encode([self.thr] * n, 99)

    def ref_step(self, R, SR, chain_r, inp, threads):
        cts, ct_t = inp
        return R.threshold_count_pool(SR.ev, cts, ct_t, self.spec.norm, chain_r, SR.keys, self.spec.slots,
                                      threads, False)[0]

    def gpu_ladder(self, blocks):
        cts = [self.client[self.mine.index(b)] for b in blocks]
        return self.partial(cts + [self.client[-1]], len(cts), self.G.PolyEval.ladder)


class Statement:
    """Configs 4/5: the full TETRIS statement per record block (linear risk
    score, three private thresholds, AND, plaintext flag), summed."""
    metric = "encrypted records/sec per TETRIS query (full statement; amortized us/record in config)"
    slot_sum = True

    def check(self, res):
        return decrypted_count(self.G, self.S, self.spec, res, self.plain_count())

    def __init__(self, G, W, spec, rank=0, world=1, rotations=True, device=True):
        from paper_2412_13269_b200 import distributed as D
        self.G, self.W, self.spec = G, W, spec
        self.batched, self.max_blocks = True, 8
        self.d = W.statement_data(spec)
        if not device:  # inputs only (the CPU reference arm)
            return
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

    def partial(self, client, streams, mode, ready=None):
        if not self.blocks:
            return None
        q, bl = self._bind(client, self.blocks)
        thr = self.W.threshold_fn(self.S, self.chain, mode)
        if self.batched:  # blocks as ciphertext batches (shared launches and key reads)
            return self.W.statement_partial_batched(self.S, q, bl, thr, streams=streams, max_blocks=self.max_blocks,
                                                    ready=ready)
        if ready:
            for name in self.upload_groups:
                ready(name)
        return self.W.statement_partial(self.S, q, bl, thr, streams)

    def plain_count(self):
        return self.W.statement_plain_count(self.d)

    def ref_inputs(self, R, SR, chain_r, host_encode, blocks):
        from types import SimpleNamespace as NS
        W, d, n, L = self.W, self.d, self.spec.slots, SR.ring.max_level()
        ct_w = [host_encode([wj] * n, 400 + j) for j, wj in enumerate(d.w)]
        ct_t = [host_encode([tk] * n, 90 + k) for k, tk in enumerate(d.t)]
        out = []
        for b in blocks:
            sl = slice(b * n, (b + 1) * n)
            pts, sc = W.encode_plaintexts(SR, [d.attrs[sl, j] for j in range(8)] + [d.flag[sl]], L)
            out.append(NS(ct_sugar=host_encode(d.sugar[sl], 200 + b), ct_bp=host_encode(d.bp[sl], 300 + b),
                          pt_attr=pts[:8], attr_scale=sc, pt_flag=pts[8], flag_scale=sc))
        return NS(ct_w=ct_w, ct_t=ct_t), out

    def ref_step(self, R, SR, chain_r, inp, threads):
        """The reference's own code path, threads over blocks x thresholds;
        per block the same ops as workloads.statement_block."""
        from concurrent.futures import ThreadPoolExecutor
        W, ev, keys = self.W, SR.ev, SR.keys
        q, blocks = inp

        def thr(x, t, norm):
            return R.eval_private_threshold_plain_norm(ev, x, t, norm, chain_r, keys)

        with ThreadPoolExecutor(max(1, threads)) as ex:
            risks = list(ex.map(lambda b: W.linear_score(SR, q.ct_w, b.pt_attr, b.attr_scale), blocks))
            futs = [(ex.submit(thr, b.ct_sugar, q.ct_t[0], 1.0), ex.submit(thr, b.ct_bp, q.ct_t[1], 1.0),
                     ex.submit(thr, r, q.ct_t[2], W.RISK_NORM)) for b, r in zip(blocks, risks)]
            outs = []
            for b, (f1, f2, f3) in zip(blocks, futs):
                a = ev.rescale(ev.mul_relin(f1.result(), f2.result(), keys))
                a = ev.rescale(ev.mul_relin(a, f3.result(), keys))
                outs.append(ev.rescale(ev.mul_plain(a, b.pt_flag, b.flag_scale)))
        acc = outs[0]
        for o in outs[1:]:
            acc = ev.add(acc, o)
        return acc

    def gpu_ladder(self, blocks):
        q, bl = self._bind(self.client, self.blocks)
        sel = [bl[self.mine.index(b)] for b in blocks]
        thr = self.W.threshold_fn(self.S, self.chain, self.G.PolyEval.ladder)
        if self.batched:  # the product path, in ladder mode
            return self.W.statement_partial_batched(self.S, q, sel, thr, streams=2, max_blocks=self.max_blocks)
        return self.W.statement_partial(self.S, q, sel, thr, len(sel))


class LinearScore:
    """Config 2: encrypted linear score per record block, sum_j mul_plain(
    Enc(w_j), pt(attr_j)) + rescale (8 pt x ct MACs); plaintext attributes
    resident on the server, the 8 weight ciphertexts are the query."""
    metric = "encrypted records/sec per linear-score query (8 pt x ct MACs + rescale per block)"
    slot_sum = False

    def __init__(self, G, W, spec, rank=0, world=1, rotations=True, device=True):
        from paper_2412_13269_b200 import distributed as D
        self.G, self.W, self.spec = G, W, spec
        self.batched, self.max_blocks = True, 8
        self.attrs, self.w = W.linear_score_data(spec)
        if not device:
            return
        self.S = W.make_context(G, spec, relin=False)
        self.chain = None
        self.mine = D.shard(spec.n_cts, world, rank)
        inp = W.config2_inputs(self.S, self.attrs, self.w)
        self.blocks = [inp.blocks[b] for b in self.mine]
        self.plain_scale = inp.plain_scale
        self.client = list(inp.ct_w)

    def partial(self, client, streams, mode):
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

    def ref_inputs(self, R, SR, chain_r, host_encode, blocks):
        from types import SimpleNamespace as NS
        W, n, L = self.W, self.spec.slots, SR.ring.max_level()
        ct_w = [host_encode([wj] * n, 400 + j) for j, wj in enumerate(self.w)]
        out = []
        for b in blocks:
            pts, sc = W.encode_plaintexts(SR, [self.attrs[b * n:(b + 1) * n, j] / W.ATTR_NORM for j in range(8)], L)
            out.append(NS(pts=pts, scale=sc))
        return ct_w, out

    def ref_step(self, R, SR, chain_r, inp, threads):
        ct_w, blocks = inp
        return [self.W.linear_score(SR, ct_w, b.pts, b.scale) for b in blocks]

    def gpu_ladder(self, blocks):
        return [self.W.linear_score(self.S, self.client, self.blocks[self.mine.index(b)], self.plain_scale)
                for b in blocks]


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

    # warm-up
    for _ in range(args.warmup):
        res = query(wl.client)
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
        ms_list, res = timed(lambda: query(wl.client), args.steps)
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

    # profiled replay of the same steps: per-kernel-class CUDA-event times
    G.profile_enable(S.ring, True)
    barrier()
    # one stream here, so every kernel's event-bracketed duration is its own
    # (concurrent streams would time-share the SMs inside the brackets)
    _, _ = timed(lambda: query(wl.client, streams=1), args.steps)
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
    dname, (dms, dn, dbytes) = dom[0], dom[1]
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
                "fp64": fp64_roofline(prof, spec.N) if dname.startswith("ntt") else None,
                "per_kernel": {k: {"ms": round(v[0] / args.steps, 4), "launches": v[1] // args.steps,
                                   "GBps": round((v[2] / v[1]) / ((v[0] / v[1]) / 1e3) / 1e9, 1)}
                               for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}}

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
        "config": {"workload": spec.name, "records": records, "N": spec.N, "levels": spec.nq - 1,
                   "q_bits": spec.q_bits, "special_primes": f"{spec.K}x{spec.sp_bits}b",
                   "dnum": -(-spec.nq // spec.group), "chain_degrees": list(spec.degrees), "alpha": spec.alpha,
                   "epsilon": spec.epsilon, "poly_eval": args.poly_eval, "streams": args.streams,
                   "batched": bool(getattr(wl, "batched", False)), "max_blocks": getattr(wl, "max_blocks", None),
                   "record_blocks": spec.n_cts, "slots": spec.slots, "secret_hw": spec.h,
                   "amortized_us_per_record": round(ms_step * 1e3 / records, 4),
                   "l2": "1 GiB buffer written between timed steps; working set (keys, blocks) > 126 MB L2",
                   "parallelism": f"block-shard x{world}", **check},
        "e2e": {"value": round(records / (e2e_ms / 1e3), 1), "unit": "records/s", "ms_per_step": round(e2e_ms, 3),
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches // args.steps),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# CPU reference: the compiled, unmodified reference (oracle/_ref)
# ---------------------------------------------------------------------------
def _ref_module():
    sys.path.insert(0, str(ROOT / "tests"))
    from common import load_ref
    return load_ref()


def _ref_setup(G, W, spec, wl, blocks, rotations=False):
    """Reference context + the workload's inputs for `blocks`, bit-identical to
    the B200 arm's (same keys/randomness streams; slot vectors encoded with the
    product's multi-threaded HOST encoder, which reproduces the reference
    Encoder's residues exactly - tests/test_host_cpu.py - instead of its
    single-threaded O(n^2) DFT)."""
    R = _ref_module()
    if R is None:
        raise RuntimeError("oracle/_ref not built")
    SR = W.make_context(R, spec, rotations=W.inner_sum_rotations(spec.slots) if rotations else [],
                        relin=bool(spec.degrees))
    sys.path.insert(0, str(ROOT / "tests"))
    from common import copy_chain
    # the B200 arm's chain when present (bit-identical, saves the host Remez
    # time of degree-63 chains), else the reference's own build_chain
    if not spec.degrees:  # no threshold in this workload
        chain_r = None
    else:
        chain_r = copy_chain(R, wl.chain) if getattr(wl, "chain", None) is not None else W.config3_chain(R, spec)
    ringG = G.RingParams(spec.N, SR.primes + SR.sp, spec.K)
    encG = G.Encoder(ringG, spec.slots)

    def encode_host(SR_, arr, scale, level):
        return [R.Poly.from_numpy(SR_.ring, encG.encode_slots_host([complex(x) for x in v], scale, level), level,
                                  R.Form.coeff, 0) for v in arr]

    SR.encode = encode_host
    lvl = SR.ring.max_level()

    def host_encode(values, label):
        m = encode_host(SR, [values], spec.delta, lvl)[0]
        return SR.ctx.encrypt(SR.sk, m, spec.delta, R.Rng(spec.seed).split(label), R.Domain.slots)

    return R, SR, chain_r, wl.ref_inputs(R, SR, chain_r, host_encode, blocks)


def ref_threads(wl, nblocks):
    """Host threads the reference uses: one per threshold job (protocol.hpp:297-311);
    the linear score is one thread (no threads in the reference's scoring)."""
    per = 3 if isinstance(wl, Statement) else (1 if isinstance(wl, ThresholdCount) else 0)
    return max(1, min(nblocks * per, os.cpu_count() or 1)) if per else 1


def cpu_baseline(G, W, spec, wl):
    """Bounded sample (~10-30 s of CPU work): the reference on one record
    block (config 3: all blocks, one thread each), compared residue for
    residue with the GPU ladder run of the same block(s)."""
    blocks = [0] if isinstance(wl, Statement) else list(range(spec.n_cts))
    R, SR, chain_r, inp = _ref_setup(G, W, spec, wl, blocks)
    threads = ref_threads(wl, len(blocks))
    t0 = time.perf_counter()
    res = wl.ref_step(R, SR, chain_r, inp, threads)
    secs = time.perf_counter() - t0
    lad = wl.gpu_ladder(blocks)
    res_l, lad_l = (res, lad) if isinstance(res, list) else ([res], [lad])
    same = all(all(np.array_equal(a.to_numpy(), b.to_numpy()) for a, b in zip(x.parts, y.parts))
               and x.scale == y.scale and x.level() == y.level() for x, y in zip(res_l, lad_l))
    recs = len(blocks) * spec.slots
    what = {ThresholdCount: "threshold", Statement: "statement ops", LinearScore: "linear score"}[type(wl)]
    return {"value": round(recs / secs, 2), "unit": "records/s", "cores": threads, "kind": "reference",
            "sample": f"{len(blocks)} record block(s) x {spec.slots} records through the reference's own "
                      f"{what} on {threads} thread(s) (unmodified headers, g++ -O2), {secs:.2f} s"
                      + ("; slot-sum not in the sample" if wl.slot_sum else ""),
            "seconds": round(secs, 2), "bit_exact_vs_gpu_ladder": bool(same),
            "note": ("reference = its own T_k-ladder polynomial evaluator; the GPU ladder run of the same blocks is "
                     "compared residue for residue (BSGS parity vs its oracle: tests/test_gpu_bsgs.py, "
                     "tests/test_gpu_statement.py)") if spec.degrees else
                    "the GPU outputs of the same blocks are compared residue for residue"}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    from paper_2412_13269_b200 import tetris as G
    from paper_2412_13269_b200 import workloads as W

    spec = W.CONFIGS[args.config]
    if _ref_module() is None:
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref not built (needs /root/reference at build time)"}))
        return
    cores = os.cpu_count() or 1
    per_block = 3 if WORKLOADS[args.config] is Statement else 1
    nblk = max(1, min(spec.n_cts, cores // per_block))
    if WORKLOADS[args.config] is LinearScore:
        nblk = spec.n_cts  # the whole (small) query
    blocks = list(range(nblk))
    t0 = time.time()

    wl = WORKLOADS[args.config](G, W, spec, device=False)
    R, SR, chain, inp = _ref_setup(G, W, spec, wl, blocks)
    threads = ref_threads(wl, nblk)
    log(f"[reference] setup {time.time() - t0:.1f}s, sample {nblk} blocks on {threads} threads")

    def step():
        t = time.perf_counter()
        wl.ref_step(R, SR, chain, inp, threads)
        return time.perf_counter() - t

    for _ in range(args.warmup):
        step()
    secs = [step() for _ in range(args.steps)]
    s = sum(secs) / len(secs)
    recs = nblk * spec.slots
    value = recs / s
    sample = (f"each step = {nblk} of {spec.n_cts} record blocks ({recs} records) through the reference's own "
              f"code path on {threads} threads (unmodified headers, g++ -O2); per-record work is identical across "
              f"blocks; the once-per-query slot-sum is not in the sample")
    print(json.dumps({
        "impl": "reference", "metric": WORKLOADS[args.config].metric,
        "value": round(value, 2), "unit": "records/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(s * 1e3, 1), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64 (mod-q RNS residues)", "data": "synthetic",
        "config": {"workload": spec.name, "records": spec.records, "N": spec.N, "levels": spec.nq - 1,
                   "sample_records": recs, "amortized_us_per_record": round(s * 1e6 / recs, 2)},
        "cpu_baseline": {"value": round(value, 2), "unit": "records/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(value, 2), "unit": "records/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
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
    ap.add_argument("--config", type=int, choices=[2, 3, 4, 5], default=4,
                    help="BASELINE.json workload: 4 = full TETRIS statement (default), 3 = threshold count, "
                         "5 = scale-out stress")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
