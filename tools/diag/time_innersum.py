"""Device time of the query tail: inner_sum over 2^15 slots (15 rotations) on
one level-2 ciphertext with the config-4 keys (the once-per-query slot sum)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import torch
from paper_2412_13269_b200 import tetris as G
from paper_2412_13269_b200 import workloads as W

spec = W.CONFIGS[4]
S = W.make_context(G, spec, rotations=W.inner_sum_rotations(spec.slots))
c = G.Ciphertext()
rng = G.Rng(3)
for lvl in (2, 4):
    c.parts = [G.sample_uniform(S.ring, lvl, 0, rng.split(i)) for i in range(2)]
    c.scale, c.domain, c.sk_id = spec.delta, G.Domain.slots, S.sk.id()
    for _ in range(3):
        G.inner_sum(S.ev, c, spec.slots, S.keys)
    S.ring.synchronize()
    ext = torch.cuda.ExternalStream(S.ring.stream_handle())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    for _ in range(10):
        G.inner_sum(S.ev, c, spec.slots, S.keys)
    e1.record(ext)
    S.ring.synchronize()
    torch.cuda.synchronize()
    print(f"inner_sum level {lvl}: {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)
    G.profile_enable(S.ring, True)
    G.inner_sum(S.ev, c, spec.slots, S.keys)
    pr = G.profile_read(S.ring)
    G.profile_enable(S.ring, False)
    print({k: (round(v[0], 3), v[1]) for k, v in pr.items()})
