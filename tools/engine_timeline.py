"""Per-CTA timeline of one engine launch in steady state (experiment build with -DQP_ENG_TIMELINE).

    python -c "from paper_2509_20214_b200 import build as b; b.build(defines=['QP_ENG_TIMELINE'],
               out='paper_2509_20214_b200/libqpalette_tl.so')"
    QP_LIB_PATH=paper_2509_20214_b200/libqpalette_tl.so python tools/engine_timeline.py --sets c2

Stamps (globaltimer ns, thread 0 of each CTA): 0 entry, 1 rotor after griddepcontrol.wait,
2 before the table store, 3 after griddepcontrol.wait / prologue, 4 first layer's x' ready,
5 main loop done, 6 exit. Printed relative to the earliest entry: min / median / max over CTAs.
"""
import ctypes as C
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import argparse
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--sets", default="c2")
    ap.add_argument("--prerotated", action="store_true")
    args = ap.parse_args()
    from paper_2509_20214_b200 import _lib as QL
    from qp_synth import activations_fp16, channel_scales, random_code_bytes
    from tests import qp_cases as Q
    from tools.engine_ab import SETS
    lib = QL.lib()
    fn = lib.qp_debug_engine_timeline
    fn.argtypes = [C.c_void_p, C.c_int]
    for name in args.sets.split(","):
        specs = SETS[name]
        cbs, rots, reps = {}, {}, []
        for r in range(3):
            lays = []
            for k, (o, i, s, x) in enumerate(specs):
                if (s, x) not in cbs:
                    cbs[(s, x)] = QL.Codebook(s, x, Q.load_fp16(s, x), L=16)
                if i not in rots:
                    rots[i] = QL.Rht(7, i)
                lays.append(QL.Layer.from_codes(random_code_bytes(Q.code_bytes(o, i, s, x), 900 + 31 * r + k),
                                                channel_scales(o, i), o, i, s, x, cbs[(s, x)], rots[i]))
            m = QL.Multi(lays)
            xs = [torch.from_numpy(activations_fp16(1, i)).cuda() for o, i, s, x in specs]
            ys = [torch.empty(1, o, device="cuda") for o, i, s, x in specs]
            reps.append((m, xs, ys, lays))
        flags = QL.QP_X_PREROTATED if args.prerotated else 0
        for it in range(12):
            m, xs, ys, _ = reps[it % 3]
            m.forward(xs, 1, ys, flags=flags)
        torch.cuda.synchronize()
        allb = np.zeros(192 * 24, dtype=np.uint64)
        assert fn(allb.ctypes.data, allb.size) == 0
        buf = allb[:192 * 8].reshape(192, 8)
        wl = allb[192 * 8:].reshape(192, 16)
        g = 148
        t = buf[:g].astype(np.int64)
        t0 = t[:, 0].min()
        names = ["entry", "rotor_wait", "pre_table", "prologue", "xready", "loop_end", "exit", "rot_done"]
        print(f"== {name} prerotated={args.prerotated}: us relative to the first CTA entry (min / median / max)")
        for k, nm in enumerate(names):
            v = t[:, k]
            v = v[v > 0]
            if len(v) == 0:
                continue
            rel = (v - t0) / 1e3
            print(f"  {nm:10s} n={len(v):3d}  {rel.min():7.2f} {statistics.median(rel):7.2f} {rel.max():7.2f}")
        le = (t[:, 5] - t0) / 1e3
        print("  loop_end per CTA (us):", " ".join(f"{v:.0f}" for v in le))
        w = (wl[:g].astype(np.int64) - t0) / 1e3                       # [cta][warp]
        rel = w - w.mean(axis=1, keepdims=True)
        print("  per-warp loop end minus the CTA mean (us), averaged over CTAs, warps 0..15:")
        print("   ", " ".join(f"{v:+.2f}" for v in rel.mean(axis=0)))
        print("  spread within a CTA (max - min), median over CTAs: %.2f us" % np.median(w.max(1) - w.min(1)))


if __name__ == "__main__":
    main()
