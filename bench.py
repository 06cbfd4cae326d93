#!/usr/bin/env python3
"""Benchmark of the B200 RNS-CKKS threshold-count query (BASELINE.json metric:
encrypted records/s & amortized us/record per TETRIS query).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One step = one full query over the workload: per-ciphertext private
threshold (composite minimax sign chain), sum of the per-ciphertext outputs,
and the log2(slots) rotate-and-add slot sum into an encrypted count.
N>1 (torchrun): ciphertexts are sharded round-robin over ranks; each rank
sums its outputs, the partial ciphertexts are NCCL-reduced to rank 0
(integer sum + mod-q fix-up kernel) and rank 0 runs the one inner_sum — the
reference's order (sum, then InnerSum; protocol.hpp:319-323), so the result
is bit-identical at every GPU count.

`--impl reference` times the reference's own CPU implementation (the
unmodified headers compiled into oracle/_ref) on the box's host cores with a
std::thread pool over ciphertexts (protocol.hpp:297-311); rank 0 only.
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
sys.path.insert(0, str(ROOT))

RECORDS_PER_CT = None  # set from the spec


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md: sample during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._thr = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.QUERY}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thr:
            self._thr.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


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

    spec = W.CONFIGS[3]
    t0 = time.time()
    rot = W.inner_sum_rotations(spec.slots) if rank == 0 else []
    S = W.make_context(G, spec, rotations=rot)
    chain = W.config3_chain(G, spec)
    scores, thr, _, _ = W.linear_scores(spec)
    from paper_2412_13269_b200 import distributed as D

    mine = D.shard(spec.n_cts, world, rank)
    D.check_exact(world, S.primes)
    cts, ct_t, _, _ = W.config3_inputs(S, ct_indices=mine, scores=scores, t=thr)
    S.ring.synchronize()
    log(f"[rank {rank}] setup {time.time() - t0:.1f}s: N={spec.N} L={spec.nq - 1} K={spec.K} cts={mine}")
    mode = G.PolyEval.bsgs if args.poly_eval == "bsgs" else G.PolyEval.ladder
    ext = torch.cuda.ExternalStream(S.ring.stream_handle(), device=torch.device("cuda", local))
    flush = torch.empty(64 << 22, dtype=torch.int32, device="cuda")  # 1 GiB > 126 MB L2

    def query(local_cts, t_ct, streams=None):
        streams = streams or args.streams
        # per-ciphertext thresholds run concurrently (one host thread + CUDA
        # stream each); outputs are summed in index order on the main stream
        acc = None
        outs = G.eval_private_threshold_plain_norm_many(S.ev, local_cts, t_ct, spec.norm, chain, S.keys,
                                                        streams, mode) if local_cts else []
        for o in outs:
            acc = o if acc is None else S.ev.add(acc, o)
        if acc is None:  # rank without ciphertexts contributes zero
            acc = S.ctx.zero_ciphertext(t_ct.level() - chain.levels_required(), 1.0, S.sk.id(), G.Domain.slots)
        if world > 1:
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
        res = query(cts, ct_t)
    barrier()
    # timed region (device-resident inputs)
    prof_region = os.environ.get("TG_PROFILE_REGION") == "1"  # ncu --profile-from-start off
    with ClockSampler(local) as clocks:
        barrier()
        if prof_region:
            torch.cuda.cudart().cudaProfilerStart()
        ms_list, res = timed(lambda: query(cts, ct_t), args.steps)
        if prof_region:
            torch.cuda.cudart().cudaProfilerStop()
        barrier()
    ms_step = sum(ms_list) / len(ms_list)
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
    _, _ = timed(lambda: query(cts, ct_t, streams=1), args.steps)
    prof = G.profile_read(S.ring)
    G.profile_enable(S.ring, False)

    # end to end through the public API: host (pinned) ciphertexts in, count out
    host_in = []
    for c in cts + [ct_t]:
        arr = G.pinned_empty([2, c.level() + 1, spec.N])
        G.ciphertext_to_numpy(c, arr)
        host_in.append((arr, c.scale, c.sk_id))
    lvl_in = ct_t.level()
    out_lvl = res.level() if rank == 0 else 0
    host_out = G.pinned_empty([2, out_lvl + 1, spec.N])

    def e2e_step():
        ups = [G.ciphertext_from_numpy(S.ring, a, lvl_in, G.Form.coeff, sc, G.Domain.slots, sid)
               for (a, sc, sid) in host_in]
        r = query(ups[:-1], ups[-1])
        if rank == 0:
            G.ciphertext_to_numpy(r, host_out)
        return r

    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    barrier()
    e2e_ms_list, _ = timed(e2e_step, args.steps)
    e2e_ms = sum(e2e_ms_list) / len(e2e_ms_list)
    if world > 1:
        tt = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    h2d = sum(a.nbytes for a, _, _ in host_in)
    d2h = host_out.nbytes if rank == 0 else 0

    # decrypt + check the count (rank 0)
    check = {}
    if rank == 0:
        enc = G.Encoder(S.ring, spec.slots)
        dec = np.array(enc.decode_slots(S.ctx.decrypt(S.sk, res), res.scale))
        count = float(dec[0].real)
        want = int((scores >= thr).sum())
        check = {"decrypted_count": round(count, 3), "plaintext_comparator_count": want}

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
    launches = sum(v[1] * (2 if k.startswith("ntt") else 1) for k, v in prof.items())
    roofline = {"bound": "hbm", "kernel": dname, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": None, "peak_kind": peak_kind,
                "bytes_per_launch": dbytes / dn, "ms_per_launch": per_launch_ms,
                "share_of_step": round(dms / total_prof_ms, 3),
                "per_kernel": {k: {"ms": round(v[0] / args.steps, 4), "launches": v[1] // args.steps,
                                   "GBps": round((v[2] / v[1]) / ((v[0] / v[1]) / 1e3) / 1e9, 1)}
                               for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            # full-size parity: the GPU ladder query vs the unmodified CPU reference
            ladder = G.eval_private_threshold_plain_norm_many(S.ev, cts, ct_t, spec.norm, chain, S.keys,
                                                              args.streams, G.PolyEval.ladder)
            lad = ladder[0]
            for o in ladder[1:]:
                lad = S.ev.add(lad, o)
            lad = G.inner_sum(S.ev, lad, spec.slots, S.keys)
            cpu = cpu_baseline(G, W, spec, S, chain, scores, thr, lad)
        except Exception as e:  # the baseline is reported, never the product
            cpu = {"value": None, "error": str(e)[:200]}

    clk = clocks.summary()
    line = {
        "metric": "encrypted records/sec per TETRIS threshold-count query (amortized us/record in config)",
        "value": round(value, 1), "unit": "records/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64 (mod-q RNS residues)", "data": "synthetic",
        "config": {"workload": spec.name, "records": records, "N": spec.N, "levels": spec.nq - 1,
                   "q_bits": spec.q_bits, "special_primes": f"{spec.K}x{spec.sp_bits}b", "dnum": -(-spec.nq // spec.group),
                   "chain_degrees": list(spec.degrees), "alpha": spec.alpha, "epsilon": spec.epsilon,
                   "poly_eval": args.poly_eval, "streams": args.streams,
                   "ciphertexts": spec.n_cts, "slots": spec.slots, "secret_hw": spec.h,
                   "amortized_us_per_record": round(ms_step * 1e3 / records, 4),
                   "l2": "1 GiB buffer written between timed steps; working set (keys) ~1.4 GB > 126 MB L2",
                   "parallelism": f"ct-shard x{world}", **check},
        "e2e": {"value": round(records / (e2e_ms / 1e3), 1), "unit": "records/s", "ms_per_step": round(e2e_ms, 3),
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# CPU baseline: the compiled, unmodified reference (oracle/_ref)
# ---------------------------------------------------------------------------
def _ref_module():
    sys.path.insert(0, str(ROOT / "tests"))
    from common import load_ref
    return load_ref()


def _ref_setup(G, W, spec, scores, thr):
    """Reference context + the same inputs (bit-identical by construction;
    slot vectors encoded once with the product's multi-threaded host encoder,
    which produces the reference encoder's exact residues)."""
    R = _ref_module()
    if R is None:
        raise RuntimeError("oracle/_ref not built")
    rot = W.inner_sum_rotations(spec.slots)
    SR = W.make_context(R, spec, rotations=rot)
    chain = W.config3_chain(R, spec)
    ringG = G.RingParams(spec.N, SR.primes + SR.sp, spec.K)
    encG = G.Encoder(ringG, spec.slots)
    lvl = SR.ring.max_level()
    n = spec.slots

    def enc(values, label):
        host = encG.encode_slots_host([complex(v) for v in values], spec.delta, lvl)
        m = R.Poly.from_numpy(SR.ring, host, lvl, R.Form.coeff, 0)
        return SR.ctx.encrypt(SR.sk, m, spec.delta, R.Rng(spec.seed).split(label), R.Domain.slots)

    cts = [enc(scores[b * n:(b + 1) * n], 100 + b) for b in range(spec.n_cts)]
    ct_t = enc([thr] * n, 99)
    return R, SR, chain, cts, ct_t


def cpu_baseline(G, W, spec, S, chain, scores, thr, gpu_result):
    R, SR, chain_r, cts, ct_t = _ref_setup(G, W, spec, scores, thr)
    threads = min(spec.n_cts, os.cpu_count() or 1)
    res, secs = R.threshold_count_pool(SR.ev, cts, ct_t, spec.norm, chain_r, SR.keys, spec.slots, threads, True)
    same = all(np.array_equal(a.to_numpy(), b.to_numpy()) for a, b in zip(res.parts, gpu_result.parts)) \
        and res.scale == gpu_result.scale and res.level() == gpu_result.level()
    return {"value": round(spec.records / secs, 2), "unit": "records/s", "cores": threads, "kind": "reference",
            "sample": f"full query: {spec.n_cts} cts x threshold on a {threads}-thread pool + sum + inner_sum "
                      f"(unmodified reference headers, g++ -O2), {secs:.1f} s",
            "seconds": round(secs, 2), "bit_exact_vs_gpu_ladder": bool(same),
            "note": "reference = its own T_k-ladder implementation; the GPU ladder query's output ciphertext "
                    "is compared residue for residue (BSGS parity vs its oracle is in tests/test_gpu_bsgs.py)"}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    from paper_2412_13269_b200 import tetris as G
    from paper_2412_13269_b200 import workloads as W

    spec = W.CONFIGS[3]
    R = _ref_module()
    if R is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference at build time)"}))
        return
    scores, thr, _, _ = W.linear_scores(spec)
    t0 = time.time()
    R, SR, chain, cts, ct_t = _ref_setup(G, W, spec, scores, thr)
    log(f"[reference] setup {time.time() - t0:.1f}s")
    threads = min(spec.n_cts, os.cpu_count() or 1)

    def step():
        return R.threshold_count_pool(SR.ev, cts, ct_t, spec.norm, chain, SR.keys, spec.slots, threads, True)[1]

    for _ in range(args.warmup):
        step()
    secs = [step() for _ in range(args.steps)]
    s = sum(secs) / len(secs)
    value = spec.records / s
    sample = (f"each step = the full query ({spec.n_cts} cts x private threshold on a {threads}-thread pool "
              f"+ sum + inner_sum), unmodified reference headers compiled g++ -O2")
    print(json.dumps({
        "impl": "reference", "metric": "encrypted records/sec per TETRIS threshold-count query (amortized us/record in config)",
        "value": round(value, 2), "unit": "records/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(s * 1e3, 1), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "u64 (mod-q RNS residues)", "data": "synthetic",
        "config": {"workload": spec.name, "records": spec.records, "N": spec.N, "levels": spec.nq - 1,
                   "amortized_us_per_record": round(s * 1e6 / spec.records, 2)},
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
    ap.add_argument("--streams", type=int, default=4, help="concurrent ciphertext pipelines per GPU")
    ap.add_argument("--poly-eval", choices=["bsgs", "ladder"], default="bsgs",
                    help="Chebyshev evaluator of the sign stages (config 3 specifies BSGS)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
