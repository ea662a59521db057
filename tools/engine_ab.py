"""Time the persistent multi-layer engine on layer sets (experiments; one JSON line per set).

    python tools/engine_ab.py [--sets c2,c2_tcq25,...] [--batch 1] [--iters 20]

Each set: enough replicas of its layers that one graph of back-to-back qp_multi_fwd launches
streams > 2x L2 of codes; events on the launching stream; reports us per launch, us per layer,
and the algorithmic GB/s (SURVEY 8(d) bytes incl. the rotation).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [(4096, 4096), (14336, 4096), (4096, 14336)]
SETS = {
    "c2": [(o, i, s, x) for o, i in SHAPES for s, x in [("tcq", 10), ("half_tcq", 13), ("tcq", 16)]],
    "c2_tcq25": [(o, i, "tcq", 10) for o, i in SHAPES] * 3,
    "c2_tcq40": [(o, i, "tcq", 16) for o, i in SHAPES] * 3,
    "c2_half325": [(o, i, "half_tcq", 13) for o, i in SHAPES] * 3,
    "big_tcq25": [(14336, 4096, "tcq", 10)] * 6,
    "sq_tcq25": [(4096, 4096, "tcq", 10)] * 9,
    "vq3": [(o, i, "vq", 12) for o, i in SHAPES] * 3,
    "nuq4": [(o, i, "nuq", 16) for o, i in SHAPES] * 3,
    "one_sq": [(4096, 4096, "tcq", 10)],
    "one_big": [(14336, 4096, "tcq", 10)],
    "one_down": [(4096, 14336, "tcq", 10)],
    "one_vq": [(4096, 4096, "vq", 12)],
    # the four launches of the C5 decoder layer (tools/decoder_layer.py --engine)
    "c5_qkv": [(4096, 4096, "half_tcq", 17), (1024, 4096, "half_tcq", 17), (1024, 4096, "half_tcq", 17)],
    "c5_o": [(4096, 4096, "nuq", 16)],
    "c5_gu": [(14336, 4096, "tcq", 12), (14336, 4096, "tcq", 12)],
    "c5_down": [(4096, 14336, "vq", 12)],
}


def c4_sets():
    """C4 (Llama-3.1-70B MLP, row-sharded at P = 1/2/4/8): rank 0's shards of gate / up (28672 x 8192)
    and down (8192 x 28672) as one engine launch -- the per-rank compute of the sharded step (the
    all-gather needs more than one GPU)."""
    out = {}
    for P in (1, 2, 4, 8):
        for s_, x4 in (("tcq", 10), ("tcq", 16), ("vq", 12), ("nuq", 16)):
            out[f"c4:p{P}:{s_}:{x4}"] = [(28672 // P, 8192, s_, x4), (28672 // P, 8192, s_, x4), (8192 // P, 28672, s_, x4)]
    return out


def palette_sets():
    """C3 through the engine: every target quantizer (2-4.5 bits) over the three C2 shapes, one
    engine launch per set (the 3 layers of one quantizer share its decode table)."""
    from tests import qp_cases as Q
    out = {}
    for s, x4 in Q.TARGET:
        out[f"c3:{s}:{x4}"] = [(o, i, s, x4) for o, i in SHAPES]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sets", default="c2,c2_tcq25,c2_tcq40,c2_half325,big_tcq25,sq_tcq25")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--prerotated", action="store_true")
    ap.add_argument("--eager", action="store_true", help="no CUDA graph (for ncu)")
    ap.add_argument("--palette", action="store_true", help="C3: every target quantizer over the C2 shapes")
    ap.add_argument("--c4", action="store_true", help="C4: 70B MLP row shards at P = 1/2/4/8 (rank 0)")
    ap.add_argument("--batches", default="")
    ap.add_argument("--per-layer", action="store_true", help="qp_linear_fwd per layer instead of qp_multi_fwd")
    ap.add_argument("--independent", action="store_true", help="QP_INDEPENDENT launches (consecutive calls overlap)")
    args = ap.parse_args()
    if args.palette:
        SETS.update(palette_sets())
        args.sets = ",".join(k for k in SETS if k.startswith("c3:"))
    if args.c4:
        SETS.update(c4_sets())
        args.sets = ",".join(k for k in SETS if k.startswith("c4:"))
    import torch
    from paper_2509_20214_b200 import _lib as QL
    from qp_synth import activations_fp16, channel_scales, random_code_bytes
    from tests import qp_cases as Q
    torch.cuda.set_device(0)
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    cbs, rots = {}, {}
    batches = [int(b) for b in args.batches.split(",")] if args.batches else [args.batch]
    for name, B in [(n, b) for n in args.sets.split(",") for b in batches]:
        specs = SETS[name]
        nbytes = sum(Q.code_bytes(o, i, s, x) for o, i, s, x in specs)
        n_rep = max(2, -(-2 * l2 // nbytes) + 1)
        multis, xs, ys = [], [], []
        alg = 0
        for o, i, s, x in specs:
            b = x / 4
            tb = Q.tlut_bits(s, x) if s in ("tcq", "half_tcq") else 0
            lut = 4 << tb if s in ("tcq", "half_tcq") else (4 << int(2 * b) if s == "vq" else 2 << int(b))
            alg += Q.code_bytes(o, i, s, x) + 4 * o + lut + 2 * B * i + 4 * B * o + (0 if args.prerotated else 4 * B * i)
        for r in range(n_rep):
            lays = []
            for k, (o, i, s, x) in enumerate(specs):
                key = (s, x)
                if key not in cbs:
                    cbs[key] = QL.Codebook(s, x, Q.load_fp16(s, x), L=16)
                if i not in rots:
                    rots[i] = QL.Rht(7, i)
                codes = random_code_bytes(Q.code_bytes(o, i, s, x), 500 + 37 * r + k)
                lays.append(QL.Layer.from_codes(codes, channel_scales(o, i), o, i, s, x, cbs[key], rots[i]))
            multis.append(QL.Multi(lays))
            xs.append([torch.from_numpy(activations_fp16(B, i)).cuda() for o, i, s, x in specs])
            ys.append([torch.empty(B, o, dtype=torch.float32, device="cuda") for o, i, s, x in specs])
        flags = (QL.QP_X_PREROTATED if args.prerotated else 0) | (QL.QP_INDEPENDENT if args.independent else 0)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            def run():
                for r in range(n_rep):
                    if args.per_layer:
                        for lay, x_, y_ in zip(multis[r].layers, xs[r], ys[r]):
                            lay.forward(x_, B, y_, flags=flags, stream=st)
                    else:
                        multis[r].forward(xs[r], B, ys[r], flags=flags, stream=st)
            run()
            st.synchronize()
            if args.eager:
                g = type("G", (), {"replay": staticmethod(run)})
            else:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    run()
            for _ in range(3):
                g.replay()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(args.iters):
                g.replay()
            b.record(st)
            b.synchronize()
        us = a.elapsed_time(b) * 1e3 / (args.iters * n_rep)
        from tools import palette as Pal
        peak, _ = Pal.hbm_peak()
        print(json.dumps({"set": name, "batch": B, "layers": len(specs), "us_per_launch": round(us, 2),
                          "us_per_layer": round(us / len(specs), 3), "gbs": round(alg / (us * 1e-6) / 1e9, 1),
                          "frac": round(alg / (us * 1e-6) / 1e9 / peak, 4), "engine_launches": multis[0].n_engine_launches,
                          "launches_per_call": multis[0].n_launches, "replicas": n_rep,
                          "prerotated": args.prerotated, "path": "per-layer" if args.per_layer else "engine", "independent": args.independent}), flush=True)
        del multis, xs, ys
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
