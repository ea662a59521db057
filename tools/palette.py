"""Palette catalog for the measurement tools (no oracle imports: the tools drive the product
library only). Widths follow Table 1 plus uniform SQ; codebook files are the frozen
fp16 tables under codebooks/."""
from __future__ import annotations

import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PALETTE = ([("tcq", x) for x in range(6, 21, 2)] + [("half_tcq", x) for x in range(7, 20, 2)]
           + [("vq", x) for x in range(6, 25, 2)] + [("nuq", x) for x in range(8, 33, 4)]
           + [("unif", x) for x in range(8, 33, 4)])
TARGET = [(s, x) for s, x in PALETTE if 8 <= x <= 18]       # north star: 2 .. 4.5 bits
C4 = [("tcq", 10), ("half_tcq", 13), ("tcq", 16), ("vq", 12), ("nuq", 16)]


def tlut_bits(scheme: str, bits_x4: int) -> int:
    b = (bits_x4 + 1) / 4 if scheme == "half_tcq" else bits_x4 / 4     # half-TCQ: upper width's LUT
    return 9 if b <= 4 else (10 if b <= 4.5 else 11)


def codebook_path(scheme: str, bits_x4: int) -> str:
    if scheme in ("tcq", "half_tcq"):
        name = f"tcq_tlut_tb{tlut_bits(scheme, bits_x4)}"
    elif scheme == "vq":
        name = f"vq_c{bits_x4 // 2}"
    else:
        name = f"{scheme}_b{bits_x4 // 4}"
    return os.path.join(ROOT, "codebooks", name + ".f16")


def load_fp16(scheme: str, bits_x4: int) -> np.ndarray:
    return np.fromfile(codebook_path(scheme, bits_x4), dtype="<f2")


def tcq_alpha(scheme: str, bits_x4: int, L: int = 16) -> float:
    """Reconstruction scale of the TCQ codebook at this width (reading R22, codebooks/tcq_alpha.json);
    1 for NUQ / UNIF / VQ."""
    if scheme not in ("tcq", "half_tcq"):
        return 1.0
    import json
    d = json.load(open(os.path.join(os.path.dirname(codebook_path("tcq", 8)), "tcq_alpha.json")))
    return float(d[f"{scheme}/{bits_x4}/L{L}"]["alpha"])


def code_bytes(d_out: int, d_in: int, scheme: str, bits_x4: int) -> int:
    return d_out * d_in * bits_x4 // 32


def lut_bytes(scheme: str, bits_x4: int) -> int:
    """Compressed codebook bytes: TCQ 2^tb x 4, VQ 2^(2b) x 4, NUQ/UNIF 2^b x 2."""
    if scheme in ("tcq", "half_tcq"):
        return 4 << tlut_bits(scheme, bits_x4)
    if scheme == "vq":
        return 4 << (bits_x4 // 2)
    return 2 << (bits_x4 // 4)


def hbm_peak() -> tuple[float, str]:
    """Roofline denominator (GB/s): MEASURED_PEAKS.json's copy bandwidth if the driver wrote it,
    else the B200_PROFILING.md fallback of 6650 GB/s (same rule as bench.py)."""
    import json
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        return float(json.load(open(pk))["hbm_gbs"]), "measured"
    return 6650.0, "fallback"
