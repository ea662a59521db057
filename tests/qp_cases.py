"""Shared test helpers: the palette catalog and frozen-codebook loading for both sides.

The frozen fp16 codebooks (codebooks/*.f16, written by scripts/build_codebooks.py from
oracle/ only) are INPUTS to both the oracle and the CUDA library; each side expands them
with its own code (oracle: quantlut_sym; library: pre-signed / pair tables in C++).
"""
from __future__ import annotations

import os

import numpy as np

from oracle import codebooks as ocb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CB_DIR = os.path.join(ROOT, "codebooks")

# (scheme, bits_x4) for every palette width of Table 1 + uniform SQ
PALETTE = (
    [("tcq", x) for x in range(6, 21, 2)]
    + [("half_tcq", x) for x in range(7, 20, 2)]
    + [("vq", x) for x in range(6, 25, 2)]
    + [("nuq", x) for x in range(8, 33, 4)]
    + [("unif", x) for x in range(8, 33, 4)]
)
# the north-star target range 2 .. 4.5 bits
TARGET = [(s, x) for s, x in PALETTE if 8 <= x <= 18]


def tlut_bits(scheme: str, bits_x4: int) -> int:
    # half-TCQ at b = mean of (b_lo, b_lo + 0.5) uses TCQ-(b_lo + 0.5)'s codebook
    b = (bits_x4 + 1) / 4 if scheme == "half_tcq" else bits_x4 / 4
    return ocb.tlut_bits_for(b)


def codebook_file(scheme: str, bits_x4: int) -> str:
    if scheme in ("tcq", "half_tcq"):
        return f"tcq_tlut_tb{tlut_bits(scheme, bits_x4)}"
    if scheme == "vq":
        return f"vq_c{bits_x4 // 2}"
    return f"{scheme}_b{bits_x4 // 4}"


def have_codebook(scheme: str, bits_x4: int) -> bool:
    return os.path.exists(os.path.join(CB_DIR, codebook_file(scheme, bits_x4) + ".f16"))


def load_fp16(scheme: str, bits_x4: int) -> np.ndarray:
    return np.fromfile(os.path.join(CB_DIR, codebook_file(scheme, bits_x4) + ".f16"), dtype="<f2")


def oracle_codebook(scheme: str, bits_x4: int, L: int = 16) -> dict:
    t = load_fp16(scheme, bits_x4).astype(np.float64)
    if scheme in ("tcq", "half_tcq"):
        return {"lut": ocb.quantlut_sym(t.reshape(-1, 2), L, tlut_bits(scheme, bits_x4)), "L": L}
    if scheme == "vq":
        return {"lut2d": t.reshape(-1, 2)}
    return {"lut": t}


def tcq_alpha(scheme: str, bits_x4: int, L: int = 16) -> float:
    """Reconstruction scale alpha of the TCQ / half-TCQ codebook at this width (reading R22,
    codebooks/tcq_alpha.json, written by scripts/calibrate_tcq_alpha.py from oracle/ only);
    1 for the other schemes."""
    if scheme not in ("tcq", "half_tcq"):
        return 1.0
    import json
    d = json.load(open(os.path.join(CB_DIR, "tcq_alpha.json")))
    return float(d[f"{scheme}/{bits_x4}/L{L}"]["alpha"])


def code_bytes(d_out: int, d_in: int, scheme: str, bits_x4: int) -> int:
    from oracle import layout
    return layout.tile_offsets(d_out, d_in, scheme, bits_x4)[1]
