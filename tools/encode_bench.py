"""GPU trellis encoder throughput (NEXT-1): qp_quantize_offline_gpu on a Llama-shaped TCQ layer.

    python tools/encode_bench.py [--shape 4096x4096] [--bits-x4 10] [--host-rows 32]

Times the GPU path end to end (host rotation + scales, GPU rotate-half Viterbi, host packing)
and, on the first --host-rows rows only, the host encoder for comparison; checks that the two
produce identical codes on those rows. W ~ N(0, 1) (seed 0).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_20214_b200 import _lib as QL  # noqa: E402
from qp_synth import gaussian_weights  # noqa: E402
from tools import palette as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="4096x4096")
    ap.add_argument("--scheme", default="tcq")
    ap.add_argument("--bits-x4", type=int, default=10)
    ap.add_argument("--host-rows", type=int, default=32)
    a = ap.parse_args()
    d_out, d_in = map(int, a.shape.split("x"))
    cb = QL.Codebook(a.scheme, a.bits_x4, P.load_fp16(a.scheme, a.bits_x4), L=16)
    r = QL.Rht(7, d_in)
    W = gaussian_weights(d_out, d_in, seed=0).astype(np.float32)
    QL.Layer.quantize_offline(W[:32], a.scheme, a.bits_x4, cb, r, gpu=True)     # warm-up (module load)
    t0 = time.perf_counter()
    lay = QL.Layer.quantize_offline(W, a.scheme, a.bits_x4, cb, r, gpu=True)
    t_gpu = time.perf_counter() - t0
    hr = a.host_rows
    t0 = time.perf_counter()
    lay_h = QL.Layer.quantize_offline(W[:hr], a.scheme, a.bits_x4, cb, r)
    t_host = time.perf_counter() - t0
    lay_g = QL.Layer.quantize_offline(W[:hr], a.scheme, a.bits_x4, cb, r, gpu=True)
    same = bool(np.array_equal(lay_h.codes(), lay_g.codes()))
    trellises = d_out * d_in // 256
    out = {"shape": a.shape, "scheme": a.scheme, "bits": a.bits_x4 / 4, "trellises": trellises,
           "gpu_seconds": round(t_gpu, 3), "gpu_trellis_per_s": round(trellises / t_gpu, 1),
           "host_rows": hr, "host_seconds": round(t_host, 3),
           "host_trellis_per_s": round(hr * d_in / 256 / t_host, 2), "host_threads": os.cpu_count(),
           "codes_identical_on_host_rows": same, "code_bytes": lay.code_bytes}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
