"""Palette sweep (BASELINE.json configs[2] "C3", and C4's 70B shapes at P=1): fused dequant-GEMV
us/launch and achieved GB/s on algorithmic bytes for every (scheme, width, shape, batch).

    python tools/sweep.py [--shapes 4096x4096,14336x4096,4096x14336] [--batches 1,2,4,8]
                          [--widths target|all] [--shards 1,2,4,8] [--out gpurun_out/sweep.jsonl]

--shards P1,...: C4 (BASELINE.json configs[3]) on one GPU: each point is the rank-0 row shard of
the layer at world size P (d_out/P contiguous rows = a byte slice of the codes, DESIGN.md section
7), timed alone; "job_gbs" = P x shard bytes / shard time, i.e. the compute side of the row-sharded
layer with every rank equally fast. The NCCL all-gather is not included (one GPU per gpurun call).

Each point: R replicas of the layer (together > 2x L2, so every launch streams from HBM), one
CUDA graph of 4R back-to-back launches (pre-rotated x, fp32 y with QP_Y_ACCUMULATE: exactly one
kernel per launch), 3 warm-up replays, 10 timed replays with CUDA events on the capturing stream.
Synthetic inputs: uniform random code bits (DESIGN.md input recipe).
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_20214_b200 import _lib as QL  # noqa: E402
from qp_synth import activations_fp16, channel_scales, random_code_bytes  # noqa: E402
from tools import palette as P  # noqa: E402


def alg_bytes(d_out, d_in, scheme, x4, batch):
    return P.code_bytes(d_out, d_in, scheme, x4) + 4 * d_out + P.lut_bytes(scheme, x4) + 2 * batch * d_in \
        + 4 * batch * d_out


def point(scheme, x4, d_out, d_in, batch, cbs, rots, l2, peak):
    key = (scheme, x4)
    if key not in cbs:
        cbs[key] = QL.Codebook(scheme, x4, P.load_fp16(scheme, x4), L=16)
    if d_in not in rots:
        rots[d_in] = QL.Rht(7, d_in)
    nb = P.code_bytes(d_out, d_in, scheme, x4)
    R = max(2, -(-2 * l2 // nb) + 1)
    s = channel_scales(d_out, d_in)
    codes = random_code_bytes(nb, 1000)       # same bits in every replica: distinct HBM addresses is what counts
    lays = [QL.Layer.from_codes(codes, s, d_out, d_in, scheme, x4, cbs[key], rots[d_in]) for i in range(R)]
    x = torch.from_numpy(activations_fp16(batch, d_in)).cuda()
    xr = torch.empty_like(x)
    rots[d_in].apply(x, batch, xr)
    y = torch.zeros(batch, d_out, device="cuda")
    fl = QL.QP_X_PREROTATED | QL.QP_Y_ACCUMULATE
    st = torch.cuda.Stream()
    n = 4 * R
    with torch.cuda.stream(st):
        for i in range(n):
            lays[i % R].forward(xr, batch, y, flags=fl, stream=st)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(n):
                lays[i % R].forward(xr, batch, y, flags=fl, stream=st)
        for _ in range(3):
            g.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(10):
            g.replay()
        b.record(st)
        b.synchronize()
    us = a.elapsed_time(b) * 1e3 / (10 * n)
    ab = alg_bytes(d_out, d_in, scheme, x4, batch)
    del lays
    return {"scheme": scheme, "bits": x4 / 4, "bits_x4": x4, "d_out": d_out, "d_in": d_in, "batch": batch,
            "us": round(us, 3), "alg_bytes": ab, "gbs": round(ab / us / 1e3, 1), "frac": round(ab / us / 1e3 / peak, 4),
            "replicas": R}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4096x4096,14336x4096,4096x14336")
    ap.add_argument("--batches", default="1,2,4,8")
    ap.add_argument("--widths", default="target")
    ap.add_argument("--schemes", default="")
    ap.add_argument("--shards", default="1")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.jsonl"))
    a = ap.parse_args()
    peak, _ = P.hbm_peak()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    widths = {"target": P.TARGET, "c4": P.C4}.get(a.widths, P.PALETTE)
    if a.schemes:
        widths = [w for w in widths if w[0] in a.schemes.split(",")]
    shapes = [tuple(map(int, s.split("x"))) for s in a.shapes.split(",")]
    batches = [int(b) for b in a.batches.split(",")]
    shards = [int(w) for w in a.shards.split(",")]
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    cbs, rots = {}, {}
    t0 = time.time()
    with open(a.out, "a") as f:
        for (d_out, d_in) in shapes:
            for scheme, x4 in widths:
                for batch in batches:
                    for world in shards:
                        r = point(scheme, x4, d_out // world, d_in, batch, cbs, rots, l2, peak)
                        if world > 1 or len(shards) > 1:
                            r.update(world=world, full_d_out=d_out, job_gbs=round(world * r["gbs"], 1),
                                     job_frac_per_gpu=r["frac"], note="rank-0 shard alone, all-gather excluded")
                        f.write(json.dumps(r) + "\n")
                        f.flush()
                        print(f'{d_out}x{d_in} P={world} {scheme:8s} {x4 / 4:5.2f}b B={batch}: {r["us"]:8.2f} us  '
                              f'{r["gbs"]:7.1f} GB/s  {100 * r["frac"]:5.1f}%', flush=True)
    print(f"sweep done in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
