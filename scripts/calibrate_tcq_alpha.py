"""Calibrate the rate-dependent TCQ scale alpha (reading R22, oracle/scaling.py); calls only oracle/.

For every TCQ width (1.5 .. 5.0 bits, L = 16, plus config C1's TCQ-2 at L = 12) and every
half-TCQ width (1.75 .. 4.75, one alpha for both halves), minimise the Gaussian distortion
D(alpha) of the rotate-half tail-biting encoder over the frozen tlut: a coarse grid, then golden
section around its best point. Common random numbers (one fixed set of N(0,1) trellis vectors)
make D(alpha) smooth in alpha. Writes codebooks/tcq_alpha.json.

    OMP_NUM_THREADS=1 python scripts/calibrate_tcq_alpha.py [--trellises 32] [--procs 8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle import codebooks as ocb  # noqa: E402
from oracle import scaling  # noqa: E402

ROOT = os.path.join(os.path.dirname(__file__), "..")
OUT = os.path.join(ROOT, "codebooks", "tcq_alpha.json")
GRID = [0.8, 0.9, 1.0, 1.1, 1.2, 1.3, 1.4, 1.5]


def tlut(tb: int) -> np.ndarray:
    return np.fromfile(os.path.join(ROOT, "codebooks", f"tcq_tlut_tb{tb}.f16"), dtype="<f2") \
        .astype(np.float64).reshape(-1, 2)


def jobs():
    """(key, scheme, bits_x4, L, tb, shifts): shifts = the step widths s whose distortions are
    averaged (one for TCQ, (s_lo, s_hi) for half-TCQ; the LUT is the upper width's, R12)."""
    out = []
    for x4 in range(6, 21, 2):
        b = x4 / 4
        tb = ocb.tlut_bits_for(b)
        out.append((f"tcq/{x4}/L16", "tcq", x4, 16, tb, (x4 // 2,)))
    out.append(("tcq/8/L12", "tcq", 8, 12, 9, (4,)))
    for x4 in range(7, 20, 2):
        hi = (x4 + 1) / 4
        tb = ocb.tlut_bits_for(hi)
        out.append((f"half_tcq/{x4}/L16", "half_tcq", x4, 16, tb, ((x4 - 1) // 2, (x4 + 1) // 2)))
    return out


def run(job, n_trellis: int):
    key, scheme, x4, L, tb, shifts = job
    t0 = time.time()
    lut = ocb.quantlut_sym(tlut(tb), L, tb)
    v = np.random.Generator(np.random.PCG64(4242)).standard_normal((n_trellis, 128, 2))

    def D(a):
        return float(np.mean([scaling.tcq_distortion(v, lut, s, L, a) for s in shifts]))

    grid = [(a, D(a)) for a in GRID]
    a0 = min(grid, key=lambda t: t[1])[0]
    a, d, ev = scaling.golden_min(D, a0 - 0.1, a0 + 0.1, tol=4e-3)
    unit = dict(grid)[1.0]
    return key, {"scheme": scheme, "bits_x4": x4, "L": L, "tlut_bits": tb, "shifts": list(shifts),
                 "alpha": round(a, 4), "distortion": d, "distortion_alpha1": unit,
                 "trellises": n_trellis, "vectors_seed": 4242,
                 "evals": [[round(x, 5), y] for x, y in sorted(grid + ev)], "build_s": time.time() - t0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trellises", type=int, default=32)
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 8)
    args = ap.parse_args()
    js = jobs()
    res = {}
    with Pool(args.procs) as p:
        for key, r in p.starmap(run, [(j, args.trellises) for j in js]):
            res[key] = r
            print(key, r["alpha"], r["distortion"], r["distortion_alpha1"], flush=True)
    doc = {"_about": "Rate-dependent TCQ scale alpha (reading R22, oracle/scaling.py): reconstruction "
                     "alpha * dq(r), stored scale s * alpha. Written by scripts/calibrate_tcq_alpha.py "
                     "(oracle only).", **dict(sorted(res.items()))}
    with open(OUT, "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
