"""Launch the fused dequant-GEMV for one layer a few times (for ncu / quick timing).

    python tools/prof_gemv.py --shape 14336x4096 --scheme tcq --bits-x4 10 --batch 1 --iters 5
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_20214_b200 import _lib as QL  # noqa: E402
from qp_synth import activations_fp16, channel_scales, random_code_bytes  # noqa: E402
from tools import palette as Q  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="14336x4096")
ap.add_argument("--scheme", default="tcq")
ap.add_argument("--bits-x4", type=int, default=10)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--replicas", type=int, default=0, help="layer copies cycled (0: enough for > 2x L2)")
ap.add_argument("--time", action="store_true")
ap.add_argument("--pdl", action="store_true")
ap.add_argument("--rht", action="store_true", help="forward from raw x (rotation kernel + GEMV)")
ap.add_argument("--y16", action="store_true", help="fp16 y (in-order cross-CTA reduction, no zeroing kernel)")
a = ap.parse_args()
d_out, d_in = map(int, a.shape.split("x"))
cb = QL.Codebook(a.scheme, a.bits_x4, Q.load_fp16(a.scheme, a.bits_x4), L=16)
r = QL.Rht(7, d_in)
if a.replicas <= 0:
    a.replicas = max(2, -(-2 * torch.cuda.get_device_properties(0).L2_cache_size
                          // Q.code_bytes(d_out, d_in, a.scheme, a.bits_x4)) + 1)
lays = [QL.Layer.from_codes(random_code_bytes(Q.code_bytes(d_out, d_in, a.scheme, a.bits_x4), i),
                            channel_scales(d_out, d_in), d_out, d_in, a.scheme, a.bits_x4, cb, r)
        for i in range(a.replicas)]
x = torch.from_numpy(activations_fp16(a.batch, d_in)).cuda()
xr = torch.empty_like(x)
r.apply(x, a.batch, xr)
y = torch.empty(a.batch, d_out, device="cuda", dtype=torch.float16 if a.y16 else torch.float32)
xin = x if a.rht else xr
base = 0 if a.rht else QL.QP_X_PREROTATED
for i in range(a.iters):
    lays[i % a.replicas].forward(xin, a.batch, y, flags=base | QL.QP_NO_PDL)
torch.cuda.synchronize()
if a.time:
    # back-to-back launches captured in one CUDA graph (no host gaps), replicas cycle through L2
    stream = torch.cuda.Stream()
    n = max(40, 2 * a.replicas)
    flags = base | (0 if a.pdl else QL.QP_NO_PDL)
    with torch.cuda.stream(stream):
        for i in range(n):
            lays[i % a.replicas].forward(xin, a.batch, y, flags=flags, stream=stream)
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for i in range(n):
                lays[i % a.replicas].forward(xin, a.batch, y, flags=flags, stream=stream)
    import time
    t_end = time.time() + 0.3
    while time.time() < t_end:
        g.replay()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    reps = 20
    ev[0].record(stream)
    with torch.cuda.stream(stream):
        for _ in range(reps):
            g.replay()
    ev[1].record(stream)
    torch.cuda.synchronize()
    us = ev[0].elapsed_time(ev[1]) / (reps * n) * 1e3
    nbytes = lays[0].code_bytes
    print(f"{a.shape} {a.scheme} {a.bits_x4/4}b batch {a.batch} (graph, pdl={a.pdl}, rht={a.rht}, y16={a.y16}): {us:.2f} us/launch "
          f"(incl. rotation or zero kernel), codes {nbytes/us/1e3:.1f} GB/s = {nbytes/us/1e3/6535*100:.1f}% of 6535")
