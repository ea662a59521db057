import sys, numpy as np, torch
sys.path.insert(0, '.')
from tests.test_gpu_engine import _make, TB9_MIX
from paper_2509_20214_b200 import _lib as Lb
from qp_synth import activations_fp16
items = _make(TB9_MIX)
m = Lb.Multi([it[0] for it in items])
for batch in (1, 3):
    xs = [torch.from_numpy(activations_fp16(batch, it[0].d_in, seed=11 + i)).cuda() for i, it in enumerate(items)]
    for rep in range(3):
        ys = [torch.full((batch, it[0].d_out), float("nan"), device="cuda") for it in items]
        m.forward(xs, batch, ys)
        torch.cuda.synchronize()
        for li, y in enumerate(ys):
            bad = torch.isnan(y).any(0).cpu().numpy()
            rts = sorted(set(np.nonzero(bad)[0] // 32))
            if rts: print("batch", batch, "rep", rep, "layer", li, "NaN row tiles", rts, "of", y.shape[1] // 32)
print("done")
