"""Fusion-aware mixed-scheme quantization (oracle, brute force) -- TEST INFRASTRUCTURE.

(see oracle/__init__.py). Eq. fusion_aware_msq: per Transformer block b the fusible
layer groups are G_b = {q},{k},{v},{q,k},{q,v},{k,v},{q,k,v},{o},{u},{g},{u,g},{d};
a binary P_gq selects group g fused and quantized by Q_q. Minimise sum_g sum_q P_gq sum_{l in g}
l_lq subject to (C1) every layer in exactly one active (group, quantizer) pair and (C2)
sum P_gq c_gq <= C. Data-free loss l_lq = a_l err(Q_q).

The oracle enumerates every feasible assignment (all partitions of each block's layers into
fusible groups, every quantizer per group) and keeps the best -- tiny instances only. With only
singleton groups allowed it is the plain MSQ of Eq. generic_msq.
"""
from __future__ import annotations

import itertools
import math

LAYERS = ("q", "k", "v", "o", "u", "g", "d")
GROUPS = (("q",), ("k",), ("v",), ("q", "k"), ("q", "v"), ("k", "v"), ("q", "k", "v"), ("o",), ("u",), ("g",),
          ("u", "g"), ("d",))


def block_partitions(fusion: bool = True):
    """Every way to cover the 7 layers of a block exactly once by fusible groups (C1)."""
    idx = [i for i, g in enumerate(GROUPS) if fusion or len(g) == 1]
    out = []
    for r in range(1, len(idx) + 1):
        for combo in itertools.combinations(idx, r):
            cover = [l for i in combo for l in GROUPS[i]]
            if sorted(cover) == sorted(LAYERS):
                out.append(combo)
    return out


def solve_bruteforce(a, err, cost, C, fusion=True):
    """a: [B][7] sensitivities (order q,k,v,o,u,g,d); err: [nq]; cost: [12][nq] latency of group
    type g (GROUPS order) quantized by q; C: budget. Returns (loss, cost, assignment) with
    assignment = per block a list of (group index, quantizer index), or (inf, inf, None)."""
    B, nq = len(a), len(err)
    parts = block_partitions(fusion)
    options = []                      # per block: list of (loss, cost, [(g, q), ...])
    for b in range(B):
        opts = []
        for part in parts:
            for qs in itertools.product(range(nq), repeat=len(part)):
                loss = sum(a[b][LAYERS.index(l)] * err[q] for g, q in zip(part, qs) for l in GROUPS[g])
                c = sum(cost[g][q] for g, q in zip(part, qs))
                opts.append((loss, c, list(zip(part, qs))))
        options.append(opts)
    best = (math.inf, math.inf, None)
    for pick in itertools.product(*options):
        c = sum(o[1] for o in pick)
        if c > C:
            continue
        loss = sum(o[0] for o in pick)
        if loss < best[0]:
            best = (loss, c, [o[2] for o in pick])
    return best
