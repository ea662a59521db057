"""Fusion-aware mixed-scheme quantization of Llama-3.1-8B fed by THIS library's measured kernels
(paper Eq. fusion_aware_msq, and Fig. 1's mechanism).

    python tools/plan_msq.py [--quantizers target] [--blocks 32] [--out gpurun_out/msq.jsonl]

1. err(Q): distortion of every quantizer on a 256 x 4096 N(0, 1) matrix through the product path
   (qp_quantize_offline_gpu, qp_dequantize; x' of each row by qp_rht_apply), i.e. Fig. 2 / Table 5
   measured with the B200 encoder (data-free loss a_l err(Q)).
2. c(g, Q): latency of each fusible group type of a Llama-3.1-8B block (q, k, v, qk, qv, kv, qkv,
   o, u, g, ug, d) quantized by Q: rotation + fused dequant-GEMV (qp_linear_fwd on raw x, batch 1),
   graph-timed over > 2x L2 of distinct layer copies.
3. qp_plan_msq for a sweep of latency budgets, fusion-aware and plain (singleton groups), with
   synthetic sensitivities a_l = 1 (the paper's a_l need the model and data: out of scope).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_20214_b200 import _lib as QL  # noqa: E402
from qp_synth import activations_fp16, channel_scales, gaussian_weights, random_code_bytes  # noqa: E402
from tools import palette as P  # noqa: E402

H, KV, FF = 4096, 1024, 14336
GROUP_SHAPES = [("q", H, H), ("k", KV, H), ("v", KV, H), ("qk", H + KV, H), ("qv", H + KV, H), ("kv", 2 * KV, H),
                ("qkv", H + 2 * KV, H), ("o", H, H), ("u", FF, H), ("g", FF, H), ("ug", 2 * FF, H), ("d", H, FF)]


def distortion(scheme, x4, cbs, rots, rows=256, d_in=4096):
    W = gaussian_weights(rows, d_in, seed=0).astype(np.float32)
    lay = QL.Layer.quantize_offline(W, scheme, x4, cbs[(scheme, x4)], rots[d_in], gpu=True)
    Wh = torch.empty(rows, d_in, dtype=torch.float16, device="cuda")
    lay.dequantize(Wh)
    Wg = torch.from_numpy(W).cuda().half()
    Wr = torch.empty_like(Wg)
    for r0 in range(0, rows, 8):                       # R W_j for every row (qp_rht_apply, fp16)
        rots[d_in].apply(Wg[r0:r0 + 8], 8, Wr[r0:r0 + 8])
    s = torch.from_numpy(lay.scales()).cuda()
    Wt = Wr.float() / s[:, None]
    # the stored scales are s * alpha (reading R22): the error of the unit-RMS rows is alpha^2 times
    # the error measured against W'/(s alpha)
    a = cbs[(scheme, x4)].alpha
    return float(((Wt - Wh.float()) ** 2).mean()) * a * a


def group_latency(name, d_out, d_in, scheme, x4, cbs, rots, l2):
    nb = P.code_bytes(d_out, d_in, scheme, x4)
    R = max(2, -(-2 * l2 // nb) + 1)
    s = channel_scales(d_out, d_in)
    lays = [QL.Layer.from_codes(random_code_bytes(nb, 500 + i), s, d_out, d_in, scheme, x4, cbs[(scheme, x4)],
                                rots[d_in]) for i in range(R)]
    x = torch.from_numpy(activations_fp16(1, d_in)).cuda()
    y = torch.empty(1, d_out, device="cuda")
    st = torch.cuda.Stream()
    n = 2 * R
    with torch.cuda.stream(st):
        for i in range(R):
            lays[i].forward(x, 1, y, stream=st)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(n):
                lays[i % R].forward(x, 1, y, stream=st)
        for _ in range(3):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(5):
            g.replay()
        e1.record(st)
        e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (5 * n)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quantizers", default="target")
    ap.add_argument("--blocks", type=int, default=32)
    ap.add_argument("--budgets", type=int, default=12)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "msq.jsonl"))
    a = ap.parse_args()
    qs = P.TARGET if a.quantizers == "target" else P.PALETTE
    cbs = {(s, x): QL.Codebook(s, x, P.load_fp16(s, x), L=16, alpha=P.tcq_alpha(s, x)) for s, x in qs}
    rots = {d: QL.Rht(7, d) for d in (H, FF)}
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    f = open(a.out, "w")
    err = []
    for s, x in qs:
        d = distortion(s, x, cbs, rots)
        err.append(d)
        f.write(json.dumps({"kind": "distortion", "quantizer": f"{s}-{x / 4}", "bits": x / 4, "mse": d,
                            "bound_2^-2b": 2.0 ** (-x / 2)}) + "\n")
        print(f"err {s}-{x / 4}: {d:.5f} (bound {2.0 ** (-x / 2):.5f})", flush=True)
    cost = np.zeros((12, len(qs)))
    for t, (name, d_out, d_in) in enumerate(GROUP_SHAPES):
        for j, (s, x) in enumerate(qs):
            cost[t, j] = group_latency(name, d_out, d_in, s, x, cbs, rots, l2)
            f.write(json.dumps({"kind": "latency", "group": name, "shape": [d_out, d_in], "quantizer": f"{s}-{x / 4}",
                                "us": round(cost[t, j], 3)}) + "\n")
        print(f"latency {name}: " + " ".join(f"{c:.1f}" for c in cost[t]), flush=True)
    err = np.array(err)
    B = a.blocks
    sens = np.ones((B, 7))
    lo = B * min(cost[t].min() for t in range(12)) * 4          # rough lower end; infeasible budgets are skipped
    hi = B * sum(cost[GROUP_SHAPES.index(g)].max() for g in [gs for gs in GROUP_SHAPES if len(gs[0]) == 1])
    for C in np.linspace(lo, hi, a.budgets):
        row = {"kind": "plan", "blocks": B, "budget_us": round(float(C), 2)}
        for fusion in (True, False):
            try:
                loss, c, g, q = QL.plan_msq(sens, err, cost, C, fusion)
            except QL.QPError:
                row["fusion" if fusion else "plain"] = None
                continue
            avg_bits = float(np.mean([qs[int(v)][1] / 4 for v in q[0]]))
            row["fusion" if fusion else "plain"] = {
                "loss": round(loss, 5), "latency_us": round(c, 2),
                "block0": {l: [("q", "k", "v", "qk", "qv", "kv", "qkv", "o", "u", "g", "ug", "d")[int(g[0, i])],
                               f"{qs[int(q[0, i])][0]}-{qs[int(q[0, i])][1] / 4}"] for i, l in enumerate("qkvougd")},
                "block0_mean_bits": round(avg_bits, 3)}
        f.write(json.dumps(row) + "\n")
        print(json.dumps(row), flush=True)
    f.close()


if __name__ == "__main__":
    main()
