#!/usr/bin/env python3
"""Config 1 (64 ciphertexts, 60-bit specials): one tensor+relin+rescale and one
rotation inside a cudaProfilerStart/Stop region, for an ncu launch list:
  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python tools/c1_prof.py"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2412_13269_b200 import tetris as G  # noqa: E402
from paper_2412_13269_b200 import workloads as W  # noqa: E402

spec = W.CONFIGS[1]
S, cts = bench.config1_inputs(G, W, spec, spec.n_cts)
x = G.stack_ciphertexts(cts)
y = G.stack_ciphertexts(cts[1:] + cts[:1])
for _ in range(3):
    S.ev.rescale(S.ev.mul_relin(x, y, S.keys))
    S.ev.rotate(x, 1, S.keys)
S.ring.synchronize()
torch.cuda.cudart().cudaProfilerStart()
S.ev.rescale(S.ev.mul_relin(x, y, S.keys))
S.ring.synchronize()
S.ev.rotate(x, 1, S.keys)
S.ring.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
