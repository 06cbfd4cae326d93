"""Half-BTS timing: device BootstrapEvaluator.half_bts vs
the compiled reference on one host thread, on the reference's own test
fixture shape (tests/test_gpu_bootstrap.py) at N = 256 / 1024 / 2048.
Prints one JSON line per N; residues are compared (bit_exact)."""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from common import load_ref  # noqa: E402
from test_gpu_bootstrap import _encrypt_coeffs, _fixture, _message  # noqa: E402


def main():
    from paper_2412_13269_b200 import tetris as G
    R = load_ref()
    for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "256,1024,2048").split(",")]:
        t0 = time.perf_counter()
        g = _fixture(G, 419, n=n)
        t_setup_g = time.perf_counter() - t0
        v = _message(13, n)
        cg = _encrypt_coeffs(g, v, 31)
        g["ring"].synchronize()
        g["bts"].half_bts(g["ev"], cg, g["keys"])  # warm
        g["ring"].synchronize()
        reps = 5
        t0 = time.perf_counter()
        for _ in range(reps):
            lg, rg = g["bts"].half_bts(g["ev"], cg, g["keys"])
        g["ring"].synchronize()
        t_gpu = (time.perf_counter() - t0) / reps
        line = {"N": n, "gpu_ms": round(t_gpu * 1e3, 3), "gpu_setup_s": round(t_setup_g, 2)}
        if R is not None:
            t0 = time.perf_counter()
            r = _fixture(R, 419, n=n)
            line["ref_setup_s"] = round(time.perf_counter() - t0, 2)
            cr = _encrypt_coeffs(r, v, 31)
            t0 = time.perf_counter()
            lr, rr = r["bts"].half_bts(r["ev"], cr, r["keys"])
            line["ref_ms_1thread"] = round((time.perf_counter() - t0) * 1e3, 1)
            line["bit_exact"] = bool(all(np.array_equal(a.to_numpy(), b.to_numpy())
                                         for x, y in ((lg, lr), (rg, rr)) for a, b in zip(x.parts, y.parts)))
            line["speedup"] = round(line["ref_ms_1thread"] / line["gpu_ms"], 1)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
