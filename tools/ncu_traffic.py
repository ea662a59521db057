"""Per-launch DRAM traffic of the fused GEMV for the bench workload (roofline `traffic`).

On the GPU box (one GPU, under ncu):
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        -k regex:qp_gemv_kernel --print-units base --csv --log-file gpurun_out/traffic.csv python tools/ncu_traffic.py
Here:
    python tools/ncu_traffic.py --parse gpurun_out/traffic.csv   -> profiles/gemv_traffic.json
Every bench layer is launched twice (pre-rotated x, fp32 y with QP_Y_ACCUMULATE, as bench.py's
kernel timing does); the second launch of each layer is the one recorded.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def launch():
    import numpy as np
    import torch

    import bench
    from paper_2509_20214_b200 import _lib as QL
    from qp_synth import activations_fp16, channel_scales, random_code_bytes
    batch = int(os.environ.get("QP_BATCH", "1"))
    for L in bench.workload(1):
        cb = QL.Codebook(L["scheme"], L["bits_x4"], np.fromfile(bench.tlut_file(L["scheme"], L["bits_x4"])[0],
                                                                 dtype="<f2"), L=16)
        r = QL.Rht(bench.SEED, L["d_in"])
        lay = QL.Layer.from_codes(random_code_bytes(bench.code_bytes(L["d_out"], L["d_in"], L["bits_x4"]), 0),
                                  channel_scales(L["d_out"], L["d_in"]), L["d_out"], L["d_in"], L["scheme"],
                                  L["bits_x4"], cb, r)
        x = torch.from_numpy(activations_fp16(batch, L["d_in"])).cuda()
        xr = torch.empty_like(x)
        r.apply(x, batch, xr)
        y = torch.zeros(batch, L["d_out"], device="cuda")
        for _ in range(2):
            lay.forward(xr, batch, y, flags=QL.QP_X_PREROTATED | QL.QP_Y_ACCUMULATE | QL.QP_NO_PDL)
        torch.cuda.synchronize()
        print(f'{L["d_out"]}x{L["d_in"]}:{L["scheme"]}:{L["bits_x4"]}:b{batch}', flush=True)


def parse(csv_path, batch=1):
    import csv
    import bench
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = {}
    for r in rows[1:]:
        per.setdefault(int(r[ii]), {})[r[mi]] = float(r[vi].replace(",", ""))
    ids = sorted(per)
    layers = bench.workload(1)
    assert len(ids) == 2 * len(layers), (len(ids), len(layers))
    out = {"source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum ({os.path.basename(csv_path)}), "
                     "second launch of each layer", "layers": {}}
    for i, L in enumerate(layers):
        m = per[ids[2 * i + 1]]
        alg = bench.layer_bytes(L["d_out"], L["d_in"], L["bits_x4"], L["tb"], batch)[0]
        rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
        out["layers"][f'{L["d_out"]}x{L["d_in"]}:{L["scheme"]}:{L["bits_x4"]}:b{batch}'] = {
            "dram_bytes": rd + wr, "algorithmic_bytes": alg, "ratio": round((rd + wr) / alg, 4),
            "duration_ns": m.get("gpu__time_duration.sum")}
    return out


def launch_engine(batches=(1, 8)):
    """The bench step through the engine (one qp_multi_fwd launch over the 9 C2 layers, raw x:
    rotation jobs included), 3 launches per batch size, no PDL (serialised under ncu)."""
    import numpy as np
    import torch

    import bench
    from paper_2509_20214_b200 import _lib as QL
    from qp_synth import activations_fp16, channel_scales, random_code_bytes
    lays, cbs, rots = [], {}, {}
    for li, L in enumerate(bench.workload(1)):
        key = (L["scheme"], L["bits_x4"])
        if key not in cbs:
            cbs[key] = QL.Codebook(L["scheme"], L["bits_x4"], np.fromfile(bench.tlut_file(*key)[0], dtype="<f2"), L=16)
        if L["d_in"] not in rots:
            rots[L["d_in"]] = QL.Rht(bench.SEED, L["d_in"])
        lays.append(QL.Layer.from_codes(random_code_bytes(bench.code_bytes(L["d_out"], L["d_in"], L["bits_x4"]), li),
                                        channel_scales(L["d_out"], L["d_in"]), L["d_out"], L["d_in"], L["scheme"],
                                        L["bits_x4"], cbs[key], rots[L["d_in"]]))
    m = QL.Multi(lays)
    for batch in batches:
        xs = [torch.from_numpy(activations_fp16(batch, l.d_in)).cuda() for l in lays]
        ys = [torch.empty(batch, l.d_out, device="cuda") for l in lays]
        for _ in range(3):
            m.forward(xs, batch, ys, flags=QL.QP_NO_PDL)
        torch.cuda.synchronize()
        print(f"engine b{batch}", flush=True)


def parse_engine(csv_path, batches=(1, 8)):
    """-> profiles/engine_traffic.json: DRAM bytes of the third engine launch per batch size, tagged
    with the sha256 of the library build that ran (bench.py uses it only for that build)."""
    import csv
    import bench
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 10]
    h = rows[0]
    mi, vi, ii = h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = {}
    for r in rows[1:]:
        per.setdefault(int(r[ii]), {})[r[mi]] = float(r[vi].replace(",", ""))
    ids = sorted(per)
    assert len(ids) == 3 * len(batches), len(ids)
    out = {"source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum ({os.path.basename(csv_path)}), "
                     "third qp_engine_kernel launch of the C2 step per batch", "lib_sha256": bench.lib_sha256(),
           "dram_bytes": {}, "duration_ns": {}}
    for k, b in enumerate(batches):
        m = per[ids[3 * k + 2]]
        out["dram_bytes"][f"b{b}"] = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        out["duration_ns"][f"b{b}"] = m.get("gpu__time_duration.sum")
    return out


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--parse-engine":
        d = parse_engine(sys.argv[2])
        json.dump(d, open(os.path.join(ROOT, "profiles", "engine_traffic.json"), "w"), indent=1)
        print(json.dumps(d, indent=1))
    elif len(sys.argv) > 1 and sys.argv[1] == "--engine":
        launch_engine()
    elif len(sys.argv) > 2 and sys.argv[1] == "--parse":
        d = parse(sys.argv[2])
        json.dump(d, open(os.path.join(ROOT, "profiles", "gemv_traffic.json"), "w"), indent=1)
        print(json.dumps(d, indent=1))
    else:
        launch()
