"""Small invocations of every kernel path, for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Covers: rotation kernel, fused GEMV (atomic fp32, deterministic fp32, fp16 y, pre-rotated x,
y accumulate), x' staged in shared memory (QP_XS path via the fused rotation flag), row-pair units
(batch 8, VQ), fused groups, dequantize, the persistent multi-layer engine (qp_multi_fwd) and the
GPU trellis encoder."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_20214_b200 import _lib as QL  # noqa: E402
from qp_synth import activations_fp16, channel_scales, gaussian_weights, random_code_bytes  # noqa: E402
from tools import palette as P  # noqa: E402


def layer(scheme, x4, d_out, d_in, seed=0):
    cb = QL.Codebook(scheme, x4, P.load_fp16(scheme, x4), L=16)
    r = QL.Rht(7, d_in)
    lay = QL.Layer.from_codes(random_code_bytes(P.code_bytes(d_out, d_in, scheme, x4), seed),
                              channel_scales(d_out, d_in), d_out, d_in, scheme, x4, cb, r)
    return lay, cb, r


def main():
    torch.cuda.set_device(0)
    for scheme, x4 in (("tcq", 10), ("half_tcq", 13), ("vq", 8), ("nuq", 16)):
        lay, cb, r = layer(scheme, x4, 96, 1024)
        for batch in (1, 3, 8):
            x = torch.from_numpy(activations_fp16(batch, 1024)).cuda()
            y = torch.empty(batch, 96, device="cuda")
            lay.forward(x, batch, y)
            lay.forward(x, batch, y, flags=QL.QP_DETERMINISTIC)
            lay.forward(x, batch, y, flags=QL.QP_FUSE_RHT)
            lay.forward(x, batch, y, flags=QL.QP_Y_ACCUMULATE)
            y16 = torch.empty(batch, 96, device="cuda", dtype=torch.float16)
            lay.forward(x, batch, y16)
            xr = torch.empty_like(x)
            r.apply(x, batch, xr)
            lay.forward(xr, batch, y, flags=QL.QP_X_PREROTATED)
        W = torch.empty(96, 1024, dtype=torch.float16, device="cuda")
        lay.dequantize(W)
    # row pairs (batch 8, small table) with several CTAs sharing row tiles
    lay, cb, r = layer("vq", 12, 256, 2048)
    x = torch.from_numpy(activations_fp16(8, 2048)).cuda()
    lay.forward(x, 8, torch.empty(8, 256, device="cuda"))
    # fused group
    cb = QL.Codebook("tcq", 12, P.load_fp16("tcq", 12), L=16)
    r = QL.Rht(7, 512)
    ms = [QL.Layer.from_codes(random_code_bytes(P.code_bytes(d, 512, "tcq", 12), i), channel_scales(d, 512), d, 512,
                              "tcq", 12, cb, r) for i, d in enumerate((64, 32, 32))]
    g = QL.Group(ms)
    x = torch.from_numpy(activations_fp16(2, 512)).cuda()
    g.forward(x, 2, [torch.empty(2, d, device="cuda") for d in (64, 32, 32)])
    # persistent multi-layer engine: tb = 9 family (rotation jobs with 1 and 7 Hadamard blocks, split
    # row tiles through the self-cleaning workspace, fp32 / fp16 / accumulate), a VQ group, a fallback
    specs = [("tcq", 10, 96, 1024), ("half_tcq", 13, 64, 1024), ("tcq", 16, 32, 3584), ("vq", 12, 64, 512),
             ("unif", 32, 32, 256)]
    eng = [layer(s_, x_, o_, i_, seed=50 + k) for k, (s_, x_, o_, i_) in enumerate(specs)]
    m = QL.Multi([e[0] for e in eng])
    for batch in (1, 3, 8):
        xs = [torch.from_numpy(activations_fp16(batch, i_)).cuda() for (_, _, _, i_) in specs]
        ys = [torch.empty(batch, o_, device="cuda") for (_, _, o_, _) in specs]
        m.forward(xs, batch, ys)
        m.forward(xs, batch, ys, flags=QL.QP_Y_ACCUMULATE)
        m.forward(xs, batch, [y.half() for y in ys])
    # the engine with the fused all-gather epilogue at world size 1 (peer stores, delivery, entry
    # barrier, wait kernel) over row shards of the tb = 9 layers
    shards = [e[0].shard(0, 1) for e in eng[:3]]
    m2 = QL.Multi(shards)
    pg = QL.MultiPeerGather(1, 0, [o_ for (_, _, o_, _) in specs[:3]], 2)
    for _ in range(2):
        pg.forward(m2, [torch.from_numpy(activations_fp16(2, i_)).cuda() for (_, _, _, i_) in specs[:3]])
    # GPU trellis encoder
    W = gaussian_weights(32, 256, seed=0).astype(np.float32)
    QL.Layer.quantize_offline(W, "tcq", 10, QL.Codebook("tcq", 10, P.load_fp16("tcq", 10), L=16), QL.Rht(7, 256),
                              gpu=True)
    torch.cuda.synchronize()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
