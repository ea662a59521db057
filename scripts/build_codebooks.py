"""Build and freeze every codebook the GPU path loads (calls only oracle/ and qp_synth/).

Writes codebooks/<name>.f16 (little-endian IEEE fp16, row-major) and codebooks/MANIFEST.json
(sha256, construction, sample count, seed, held-out distortion). The fp16 bytes are then
normative for both the oracle and the CUDA library (reading R7).

  python scripts/build_codebooks.py [--only tcq|nuq|unif|vq] [--vq-max-c 10]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle import codebooks as cb  # noqa: E402
from qp_synth import gaussian_vectors  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "codebooks")
N_TRAIN = 1 << 20


def write(name: str, arr16: np.ndarray, meta: dict, manifest: dict) -> None:
    path = os.path.join(OUT, name + ".f16")
    data = np.ascontiguousarray(arr16.astype("<f2")).tobytes()
    with open(path, "wb") as f:
        f.write(data)
    meta.update({"file": name + ".f16", "bytes": len(data), "sha256": hashlib.sha256(data).hexdigest(),
                 "shape": list(arr16.shape)})
    manifest[name] = meta
    print(name, meta.get("distortion_holdout"), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="all")
    ap.add_argument("--vq-max-c", type=int, default=10)
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    mpath = os.path.join(OUT, "MANIFEST.json")
    manifest = json.load(open(mpath)) if os.path.exists(mpath) else {}
    hold = gaussian_vectors(1 << 20, 2, seed=99)
    if args.only in ("all", "nuq"):
        for b in range(1, 9):
            lv = cb.freeze_fp16(cb.nuq_lloyd_max(b))
            q = np.asarray(lv, np.float64)[np.argmin(np.abs(hold[:, :1] - np.asarray(lv, np.float64)[None, :]), axis=1)]
            write(f"nuq_b{b}", lv, {"kind": "nuq", "bits": b, "construction": "Lloyd-Max, exact Gaussian integrals (P:981-982 population limit)",
                                    "mse_exact_f64": cb.scalar_mse(cb.nuq_lloyd_max(b)),
                                    "distortion_holdout": float(np.mean((hold[:, 0] - q) ** 2))}, manifest)
    if args.only in ("all", "unif"):
        for b in range(2, 9):
            lv, d = cb.unif_optimal(b)
            lv16 = cb.freeze_fp16(lv)
            write(f"unif_b{b}", lv16, {"kind": "unif", "bits": b, "delta": d,
                                       "construction": "MSE-optimal symmetric uniform grid (reading R15)",
                                       "mse_exact_f64": cb.scalar_mse(lv)}, manifest)
    if args.only in ("all", "tcq"):
        for tb in (9, 10, 11):
            t0 = time.time()
            tl = cb.freeze_fp16(cb.tcq_tlut(tb, gaussian_vectors(N_TRAIN, 2, seed=200 + tb), seed=tb))
            write(f"tcq_tlut_tb{tb}", tl, {"kind": "tcq_tlut", "tlut_bits": tb, "samples": N_TRAIN, "seed": 200 + tb,
                                           "construction": "sklearn Lloyd k-means (max_iter 300, tol 1e-6) + unit 2nd-moment scale (P:1022-1023, reading R6)",
                                           "second_moment": float(np.mean(np.asarray(tl, np.float64) ** 2)),
                                           "build_s": time.time() - t0}, manifest)
    if args.only in ("all", "vq"):
        for c in range(3, args.vq_max_c + 1):
            t0 = time.time()
            v = cb.freeze_fp16(cb.vq_codebook(c / 2, gaussian_vectors(N_TRAIN, 2, seed=300 + c), seed=c))
            vf = np.asarray(v, np.float64)
            idx = np.concatenate([np.argmin(((hold[i:i + 65536, None, :] - vf[None]) ** 2).sum(-1), axis=1)
                                  for i in range(0, hold.shape[0], 65536)])
            dist = float(np.mean(((hold - vf[idx]) ** 2).sum(-1)) / 2)
            write(f"vq_c{c}", v, {"kind": "vq", "bits": c / 2, "samples": N_TRAIN, "seed": 300 + c,
                                  "construction": "sklearn Lloyd k-means, max_iter 300, tol 1e-6 (P:1000-1001)",
                                  "distortion_holdout": dist, "build_s": time.time() - t0}, manifest)
    with open(mpath, "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
