"""Benchmark of the Q-Palette fused dequant-GEMV hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N ... bench.py --gpus N    (row-sharded layers + NCCL all-gather)

Workload (BASELINE.json configs[1], "C2"): the Llama-3.1-8B layer shapes (d_out, d_in) =
(4096, 4096), (14336, 4096), (4096, 14336), each at TCQ 2.5 / half-TCQ 3.25 / TCQ 4.0 bits
(L = 16), batch 1, synthetic uniform-random codes (= Gaussianized weights, DESIGN.md input
recipe), x ~ N(0,1) fp16. One step = for each of the 9 layers: the activation rotation
kernel + the fused dequant-GEMV kernel (qp_linear_fwd), captured once in a CUDA graph.
Metric: achieved HBM GB/s on the algorithmic (compressed) bytes of the step, plus us/layer.
Two replicas of every layer alternate between steps (326 MB > 126 MB L2: inputs larger
than L2). With N > 1 every layer is row-sharded over the ranks and each forward ends with
an NCCL all-gather of y (strong scaling; total work fixed).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("fused dequant-GEMV µs/layer and achieved HBM GB/s vs ~8 TB/s, batch 1–8, 1/2/4/8 B200")
SHAPES = [(4096, 4096), (14336, 4096), (4096, 14336)]
WIDTHS = [("tcq", 10), ("half_tcq", 13), ("tcq", 16)]
BATCH = 1
SEED = 7
REPLICAS = 2


def tlut_file(scheme: str, bits_x4: int) -> str:
    b = (bits_x4 + 1) / 4 if scheme == "half_tcq" else bits_x4 / 4     # half-TCQ: upper width's tlut
    tb = 9 if b <= 4 else (10 if b <= 4.5 else 11)
    return os.path.join(ROOT, "codebooks", f"tcq_tlut_tb{tb}.f16"), tb


def code_bytes(d_out: int, d_in: int, bits_x4: int) -> int:
    return d_out * d_in * bits_x4 // 32


def layer_bytes(d_out, d_in, bits_x4, tb, batch):
    """Algorithmic bytes: codes + fp32 scales + compressed LUT + x' in + y out."""
    gemv = code_bytes(d_out, d_in, bits_x4) + 4 * d_out + (4 << tb) + 2 * batch * d_in + 4 * batch * d_out
    rht = 4 * batch * d_in            # read x fp16, write x' fp16
    return gemv, rht


def workload(world=1):
    out = []
    for d_out, d_in in SHAPES:
        for scheme, x4 in WIDTHS:
            _, tb = tlut_file(scheme, x4)
            out.append(dict(d_out=d_out, d_in=d_in, scheme=scheme, bits_x4=x4, tb=tb, m=d_out // world))
    return out


class Clocks:
    """SM clock and throttle-reason sampling DURING the timed region (B200_PROFILING.md clocks
    line), through NVML from a background thread every 2 ms (nvidia-smi -lms into a pipe is
    block-buffered and returned nothing for short regions)."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, index: int):
        self.index, self.sm, self.reasons, self.max_mhz = index, [], set(), None
        self.stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            masks = {k: getattr(N, v) for k, v in self.REASONS.items()}

            def run():
                while not self.stop.is_set():
                    self.sm.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                    r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.reasons.update(k for k, m in masks.items() if r & m)
                    time.sleep(0.002)
            self.t = threading.Thread(target=run, daemon=True)
            self.t.start()
        except Exception:                      # no NVML: report no samples
            self.t = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


def ncu_traffic(layers, batch):
    """DRAM bytes (read + write) per GEMV launch, averaged over the step's layers, from the
    committed ncu capture (profiles/gemv_traffic.json, written by tools/ncu_traffic.py --parse);
    None if that capture does not cover this workload."""
    p = os.path.join(ROOT, "profiles", "gemv_traffic.json")
    if not os.path.exists(p):
        return None, None
    d = json.load(open(p))
    vals = []
    for L in layers:
        k = f'{L["m"]}x{L["d_in"]}:{L["scheme"]}:{L["bits_x4"]}:b{batch}'
        if k not in d["layers"]:
            return None, None
        vals.append(d["layers"][k]["dram_bytes"])
    return sum(vals) / len(vals), d.get("source")


def lib_sha256() -> str:
    import hashlib
    with open(os.path.join(ROOT, "paper_2509_20214_b200", "libqpalette.so"), "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def engine_traffic(batch):
    """DRAM bytes (read + write) per engine launch from the ncu capture in
    profiles/engine_traffic.json (tools/ncu_traffic.py --engine), used only if that capture was taken
    with THIS library build (sha256 of libqpalette.so) and this batch; else (None, why)."""
    p = os.path.join(ROOT, "profiles", "engine_traffic.json")
    if not os.path.exists(p):
        return None, "no capture (profiles/engine_traffic.json)"
    d = json.load(open(p))
    if d.get("lib_sha256") != lib_sha256():
        return None, "capture is of another build (lib sha256 differs)"
    v = d.get("dram_bytes", {}).get(f"b{batch}")
    return (v, d.get("source")) if v else (None, f"no capture at batch {batch}")


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def oracle_sample(layers, budget_rows=512, which=None):
    """CPU baseline: the float64 oracle (decode + RHT + matvec) on a bounded sample: the first
    `budget_rows` rows of every layer (or of layers[which] only)."""
    import oracle.decode as odec
    import oracle.rht as orht
    from oracle import codebooks as ocb
    from qp_synth import activations_fp16, channel_scales, random_code_bytes
    total_bytes, t0 = 0, time.perf_counter()
    for li, L in enumerate(layers):
        if which is not None and li != which:
            continue
        d_out, d_in, scheme, x4, tb = L["d_out"], L["d_in"], L["scheme"], L["bits_x4"], L["tb"]
        tl = np.fromfile(tlut_file(scheme, x4)[0], dtype="<f2").astype(np.float64).reshape(-1, 2)
        book = {"lut": ocb.quantlut_sym(tl, 16, tb), "L": 16}
        rows = min(budget_rows, d_out)
        nb = code_bytes(rows, d_in, x4)
        codes = random_code_bytes(nb, li)
        x = activations_fp16(BATCH, d_in).astype(np.float64)
        s = channel_scales(d_out, d_in)[:rows]
        W = odec.decode_layer(codes, rows, d_in, scheme, x4, book)
        y = (orht.rht_apply(x, SEED) @ W.T) * s[None, :]
        assert np.isfinite(y).all()
        g, r = layer_bytes(rows, d_in, x4, tb, BATCH)
        total_bytes += g + r
    dt = time.perf_counter() - t0
    return total_bytes, dt


def cpu_info():
    """CPU model, logical CPUs and the BLAS / OpenMP thread pools (threadpoolctl) of this process."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    pools = []
    try:
        from threadpoolctl import threadpool_info
        pools = [{"api": i.get("user_api"), "lib": i.get("internal_api"), "threads": i.get("num_threads")}
                 for i in threadpool_info()]
    except Exception:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "thread_pools": pools}


# On-chip ceilings of the fused dequant-GEMV, per weight pair: issue slots of the
# decode + MMA (from the engine's SASS: TCQ SHF + 2 IMAD + LOP3 + LDS + HMMA/4 + code loads ~ 5.3;
# VQ / NUQ SHF + LOP3 + LDS + HMMA/4 ~ 3.3) at 4 warp-instructions / clk / SM, and one shared-memory
# LUT wavefront per 32 pairs (1 wavefront / clk / SM).
ISSUE_PER_PAIR = {"tcq": 5.3, "half_tcq": 5.3, "vq": 3.3, "nuq": 3.3, "unif": 3.3}


def ceilings(layers, batch, peak_gbs, sm_mhz, n_sm=148):
    """Fractions of the HBM roofline the step could reach if bound by issue slots, by shared-memory
    LUT wavefronts, or by the slower of the two per layer (time-weighted over the step)."""
    f = (sm_mhz or 1965.0) * 1e6
    t_hbm = t_issue = t_smem = t_all = 0.0
    nbytes = 0
    for L in layers:
        g, r = layer_bytes(L["d_out"], L["d_in"], L["bits_x4"], L["tb"], batch)
        pairs = L["d_out"] * L["d_in"] / 2
        th = (g + r) / (peak_gbs * 1e9)
        ti = pairs * ISSUE_PER_PAIR[L["scheme"]] / (128.0 * n_sm * f)
        ts = pairs / (32.0 * n_sm * f)
        t_hbm += th
        t_issue += max(th, ti)
        t_smem += max(th, ts)
        t_all += max(th, ti, ts)
        nbytes += g + r
    return {"issue_frac": round(t_hbm / t_issue, 4), "smem_frac": round(t_hbm / t_smem, 4),
            "frac": round(t_hbm / t_all, 4), "sm_mhz": sm_mhz,
            "model": "per layer max(HBM bytes / peak, pairs x issue-slots-per-pair / (4 warp-instr/clk x 32 x "
                     "148 SMs), pairs / (32/clk x 148 SMs)); issue slots per pair from the engine SASS "
                     "(TCQ 5.3, VQ/NUQ 3.3)"}


def cpu_cores():
    try:
        from threadpoolctl import threadpool_info
        th = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        th = os.cpu_count() or 1
    return th


def run_reference(args, rank, world):
    """--impl reference: the float64 oracle as it stands, on the host cores. Each step is a
    bounded sample of the C2 workload: one 32-row tile of one layer, cycling through the 9
    layers (so K steps stay within minutes at the default K)."""
    if rank != 0:
        return
    layers = workload(1)
    times, nbytes = [], []
    for i in range(args.warmup + args.steps):
        nb, dt = oracle_sample(layers, budget_rows=32, which=i % len(layers))
        if i >= args.warmup:
            times.append(dt)
            nbytes.append(nb)
    t = sum(times) / len(times)
    v = sum(nbytes) / sum(times) / 1e9
    cores = cpu_cores()
    sample = "one 32-row tile of one C2 layer per step, cycling through the 9 layers: float64 decode + RHT + matvec"
    line = {"metric": METRIC, "value": round(v, 6), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": "C2: Llama-3.1-8B (4096x4096, 14336x4096, 4096x14336) x TCQ-2.5 / half-TCQ-3.25 / "
                                   "TCQ-4.0 (L=16), batch 1 (bounded CPU sample, see cpu_baseline.sample)",
                       "batch": BATCH},
            "cpu_baseline": {"value": round(v, 6), "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": round(v, 6), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--allgather", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1: p2p = the all-gather fused into the engine epilogue (peer stores over NVLink, "
                         "qp_multi_fwd_sharded_p2p; default); nccl = engine + one grouped ncclAllGather")
    ap.add_argument("--path", default="engine", choices=["engine", "layer"],
                    help="engine: one persistent qp_multi_fwd launch per step (default); layer: qp_linear_fwd "
                         "per layer (rotation kernel + GEMV kernel each)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2509_20214_b200 import _lib as QL
    from qp_synth import activations_fp16, channel_scales, random_code_bytes

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # the row-sharded (N > 1) path; QP_BENCH_FORCE_SHARDED=1 runs it at N = 1 (row shard x1, NCCL and the
    # fused all-gather at world size 1) -- a check of this code path on a one-GPU box, not a bench line
    sharded = world > 1 or os.environ.get("QP_BENCH_FORCE_SHARDED") == "1"
    if sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    batch = args.batch
    layers = workload(world)
    cbs = {}
    for L in layers:
        key = (L["scheme"], L["bits_x4"])
        if key not in cbs:
            cbs[key] = QL.Codebook(L["scheme"], L["bits_x4"], np.fromfile(tlut_file(*key)[0], dtype="<f2"), L=16)
    rots = {d_in: QL.Rht(SEED, d_in) for _, d_in in SHAPES}
    comm = None
    if sharded:
        uid = [QL.NcclComm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = QL.NcclComm(uid[0], world, rank)

    # layers (replicas x 9), each rank holding its row shard
    insts = []
    for rep in range(REPLICAS):
        for li, L in enumerate(layers):
            d_out, d_in = L["d_out"], L["d_in"]
            codes = random_code_bytes(code_bytes(d_out, d_in, L["bits_x4"]), 100 * rep + li)
            s = channel_scales(d_out, d_in)
            full = QL.Layer.from_codes(codes, s, d_out, d_in, L["scheme"], L["bits_x4"], cbs[(L["scheme"], L["bits_x4"])],
                                       rots[d_in])
            lay = full.shard(rank, world) if sharded else full
            if sharded:
                del full
            insts.append(dict(layer=lay, meta=L))
    # activations / outputs of a step live in one device buffer each (per replica), so the
    # end-to-end measurement moves a step's inputs and results with one copy each way; every
    # layer's x / y is a 256-byte-aligned view into them
    def carve(buf, sizes, elem):
        views, off = [], 0
        for n in sizes:
            views.append(buf[off:off + n])
            off += -(-n * elem // 256) * 256 // elem
        return views, off
    n_layers = len(layers)
    xs_sizes = [batch * L["d_in"] for L in layers]
    ys_sizes = [batch * L["d_out"] for L in layers]
    x_elems = carve(torch.empty(0), xs_sizes, 2)[1]
    y_elems = carve(torch.empty(0), ys_sizes, 4)[1]
    bufs = []
    for rep in range(REPLICAS):
        xb = torch.empty(x_elems, dtype=torch.float16, device=dev)
        yb = torch.empty(y_elems, dtype=torch.float32, device=dev)
        xv, _ = carve(xb, xs_sizes, 2)
        yv, _ = carve(yb, ys_sizes, 4)
        for j, L in enumerate(layers):
            inst = insts[rep * n_layers + j]
            inst["x"] = xv[j].view(batch, L["d_in"])
            inst["x"].copy_(torch.from_numpy(activations_fp16(batch, L["d_in"])))
            inst["y"] = yv[j].view(batch, L["d_out"])
        bufs.append((xb, yb))
    torch.cuda.synchronize()

    extra_flags = int(os.environ.get("QP_BENCH_FLAGS", "0"))     # experiments only (e.g. 4 = QP_DETERMINISTIC)
    use_engine = args.path == "engine"
    multis = []
    if use_engine:
        for rep in range(REPLICAS):
            multis.append(QL.Multi([inst["layer"] for inst in insts[rep * n_layers:(rep + 1) * n_layers]]))

    # N > 1, fused all-gather: every replica's y_full buffers + flags, IPC-mapped across the ranks
    pgs, allgather = [], args.allgather if (use_engine and sharded) else None
    if allgather == "p2p":
        for rep in range(REPLICAS):
            pgs.append(QL.MultiPeerGather(world, rank, [L["m"] for L in layers], batch, dtype=torch.float32))
        # one checked round before timing: the fused path must reproduce the NCCL path's y_full
        with torch.cuda.stream(torch.cuda.current_stream()):
            group = insts[:n_layers]
            multis[0].forward_sharded([i["x"] for i in group], batch, [i["y"] for i in group], comm)
            pgs[0].forward(multis[0], [i["x"] for i in group])
        torch.cuda.synchronize()
        bad = max(float((pgs[0].ys[j] - insts[j]["y"]).abs().max() / insts[j]["y"].abs().max().clamp_min(1e-30))
                  for j in range(n_layers))
        if bad > 1e-4:
            print(f"[bench] fused all-gather differs from the NCCL path ({bad:.2e}): using NCCL", file=sys.stderr)
            allgather = "nccl"

    def fwd(inst, stream=None, flags=0):
        flags |= extra_flags
        if sharded:
            inst["layer"].forward_sharded(inst["x"], batch, inst["y"], comm, flags=flags, stream=stream)
        else:
            inst["layer"].forward(inst["x"], batch, inst["y"], flags=flags, stream=stream)

    def step_fn(rep, stream):
        """One step: the 9 layers of replica `rep` (rotation + fused dequant-GEMV each)."""
        group = insts[rep * n_layers:(rep + 1) * n_layers]
        if use_engine and sharded and allgather == "p2p":
            # this rank's shards through the engine, whose epilogue stores every final value into
            # every rank's y_full (NVLink peer stores); one wait kernel for the deliveries
            pgs[rep].forward(multis[rep], [i["x"] for i in group], flags=extra_flags, stream=stream)
        elif use_engine and sharded:
            # this rank's shards through the engine, then one grouped NCCL all-gather of all 9 outputs
            multis[rep].forward_sharded([i["x"] for i in group], batch, [i["y"] for i in group], comm,
                                        flags=extra_flags, stream=stream)
        elif use_engine:
            multis[rep].forward([i["x"] for i in group], batch, [i["y"] for i in group], flags=extra_flags,
                                stream=stream)
        else:
            for inst in group:
                fwd(inst, stream)

    # ---- capture one graph per replica ------------------------------------------------
    # (QP_BENCH_EAGER=1 replays the step eagerly instead: ncu cannot profile our kernels inside
    #  captured graphs, so the launch-list profile in profiles/ is taken that way.)
    stream = torch.cuda.Stream(device=dev)
    graphs = []
    eager = os.environ.get("QP_BENCH_EAGER") == "1"

    class EagerStep:
        def __init__(self, rep):
            self.rep = rep

        def replay(self):
            with torch.cuda.stream(stream):
                step_fn(self.rep, stream)

    with torch.cuda.stream(stream):
        for rep in range(REPLICAS):
            step_fn(rep, stream)           # eager warm-up (sets kernel attributes)
        stream.synchronize()
        for rep in range(REPLICAS):
            c0 = QL.launch_count()
            if eager:
                g = EagerStep(rep)
                g.replay()
            else:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    step_fn(rep, stream)
            launches_per_step = QL.launch_count() - c0
            graphs.append(g)
    torch.cuda.synchronize()

    def barrier():
        if sharded:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        graphs[i % REPLICAS].replay()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        ev0.record(stream)
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                graphs[i % REPLICAS].replay()
        ev1.record(stream)
        ev1.synchronize()
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    if sharded:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # algorithmic bytes of one step (whole job: all ranks' shards = the full layers)
    gemv_bytes = rht_bytes = 0
    for L in layers:
        g_, r_ = layer_bytes(L["d_out"], L["d_in"], L["bits_x4"], L["tb"], batch)
        gemv_bytes += g_
        rht_bytes += r_ * world                # every rank rotates its own copy of x
    step_bytes = gemv_bytes + rht_bytes
    value = step_bytes / (ms * 1e-3) / 1e9

    # ---- per-kernel timing of the fused GEMV: one CUDA graph per layer shape/width holding
    #      back-to-back launches over the replicas (pre-rotated x, fp16 y so no zeroing kernel),
    #      timed with events on the launching stream -------------------------------------------
    xr = {}
    for inst in insts:
        d_in = inst["meta"]["d_in"]
        if d_in not in xr:
            xr[d_in] = torch.empty(batch, d_in, dtype=torch.float16, device=dev)
            rots[d_in].apply(inst["x"], batch, xr[d_in])
    # fp32 y with QP_Y_ACCUMULATE: exactly one kernel (the fused GEMV) per launch, no zeroing
    yacc = {L["d_out"]: torch.zeros(batch, L["m"], dtype=torch.float32, device=dev) for L in layers}
    kflags = QL.QP_X_PREROTATED | QL.QP_Y_ACCUMULATE
    torch.cuda.synchronize()
    per_layer_us, gemv_time_s, gemv_alg = {}, 0.0, 0
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    for li, L in enumerate(layers):
        # enough distinct copies of the layer that one graph's launches stream > 2x L2 of codes
        # (every launch reads its codes from HBM), as tools/sweep.py does
        group = [insts[rep * n_layers + li] for rep in range(REPLICAS)]
        nb = code_bytes(L["m"], L["d_in"], L["bits_x4"])
        n_copies = max(REPLICAS, -(-2 * l2 // nb) + 1)
        while len(group) < n_copies:
            src = group[len(group) % REPLICAS]["layer"]
            group.append(dict(layer=QL.Layer.from_codes(random_code_bytes(nb, 7000 + 97 * li + len(group)),
                                                        channel_scales(L["d_out"], L["d_in"])[:L["m"]], L["m"],
                                                        L["d_in"], L["scheme"], L["bits_x4"],
                                                        cbs[(L["scheme"], L["bits_x4"])], rots[L["d_in"]])))
        n_rep = 2 * len(group)
        with torch.cuda.stream(stream):
            for inst in group:
                inst["layer"].forward(xr[L["d_in"]], batch, yacc[L["d_out"]], flags=kflags, stream=stream)
            stream.synchronize()
            if eager:
                def g_replay(group=group, L=L, n_rep=n_rep):
                    for k in range(n_rep):
                        group[k % len(group)]["layer"].forward(xr[L["d_in"]], batch, yacc[L["d_out"]],
                                                             flags=kflags, stream=stream)
                g = type("G", (), {"replay": staticmethod(g_replay)})
            else:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for k in range(n_rep):
                        group[k % len(group)]["layer"].forward(xr[L["d_in"]], batch, yacc[L["d_out"]],
                                                               flags=kflags, stream=stream)
            for _ in range(3):
                g.replay()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(3, min(args.steps, 20))
            a.record(stream)
            for _ in range(reps):
                g.replay()
            b.record(stream)
            b.synchronize()
        us = a.elapsed_time(b) * 1e3 / (reps * n_rep)
        per_layer_us[f'{L["d_out"]}x{L["d_in"]}@{L["bits_x4"] / 4:g}b'] = round(us, 3)
        gemv_time_s += us * 1e-6
        gemv_alg += layer_bytes(L["m"], L["d_in"], L["bits_x4"], L["tb"], batch)[0]
    gemv_achieved = gemv_alg / gemv_time_s / 1e9
    gemv_avg_ms = gemv_time_s / n_layers * 1e3
    peak, peak_kind = measured_peaks()
    traffic, traffic_src = ncu_traffic(layers, batch)

    # ---- the engine kernel alone: one CUDA graph of back-to-back qp_multi_fwd launches alternating
    #      the two replicas (each launch streams 163 MB of codes > L2 126 MB: from HBM), events on
    #      the launching stream ---------------------------------------------------------------------
    eng = None
    eng_traffic, eng_traffic_src = engine_traffic(batch)

    def time_engine(b_):
        """us per engine launch at batch b_ (its own activations / outputs, both replicas)."""
        xs_b = [[torch.from_numpy(activations_fp16(b_, L["d_in"])).to(dev) for L in layers] for _ in range(REPLICAS)]
        ys_b = [[torch.empty(b_, L["m"], dtype=torch.float32, device=dev) for L in layers] for _ in range(REPLICAS)]
        n_rep = 8

        def launch(k):
            multis[k % REPLICAS].forward(xs_b[k % REPLICAS], b_, ys_b[k % REPLICAS], flags=extra_flags, stream=stream)
        with torch.cuda.stream(stream):
            if eager:
                def ge_replay():
                    for k in range(n_rep):
                        launch(k)
                ge = type("G", (), {"replay": staticmethod(ge_replay)})
            else:
                for k in range(REPLICAS):
                    launch(k)
                stream.synchronize()
                ge = torch.cuda.CUDAGraph()
                with torch.cuda.graph(ge, stream=stream):
                    for k in range(n_rep):
                        launch(k)
            for _ in range(3):
                ge.replay()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = max(3, min(args.steps, 30))
            a.record(stream)
            for _ in range(reps):
                ge.replay()
            b.record(stream)
            b.synchronize()
        return a.elapsed_time(b) * 1e3 / (reps * n_rep)

    # the same steps with QP_INDEPENDENT (the caller's promise that no running work touches a step's
    # x / y: consecutive steps may overlap), reported beside the dependency-safe default
    indep = None
    if use_engine and not sharded:
        gi = []
        with torch.cuda.stream(stream):
            for rep in range(REPLICAS):
                group = insts[rep * n_layers:(rep + 1) * n_layers]
                if eager:
                    gi.append(None)
                    continue
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    multis[rep].forward([i["x"] for i in group], batch, [i["y"] for i in group],
                                        flags=extra_flags | QL.QP_INDEPENDENT, stream=stream)
                gi.append(g)
            if not eager:
                for i in range(args.warmup):
                    gi[i % REPLICAS].replay()
                stream.synchronize()
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                for i in range(args.steps):
                    gi[i % REPLICAS].replay()
                a1.record(stream)
                a1.synchronize()
                ms_i = a0.elapsed_time(a1) / args.steps
                indep = {"ms_per_step": round(ms_i, 5), "value": round(step_bytes / (ms_i * 1e-3) / 1e9, 2),
                         "unit": "GB/s", "flag": "QP_INDEPENDENT"}

    batch_lines = {}
    if use_engine:
        # (N > 1: the engine alone over this rank's shards, i.e. per-rank bytes / time, no all-gather)
        eng_us = time_engine(batch)
        rank_bytes = gemv_bytes / world + rht_bytes / world
        eng = {"achieved": rank_bytes / (eng_us * 1e-6) / 1e9, "us": eng_us, "bytes": rank_bytes}
    if use_engine and not sharded:
        # the metric spans batch 1-8: the same step at the other batch sizes (engine launch alone)
        for b_ in (1, 2, 4, 8):
            if b_ == batch:
                continue
            us_b = time_engine(b_)
            bytes_b = sum(sum(layer_bytes(L["d_out"], L["d_in"], L["bits_x4"], L["tb"], b_)) for L in layers)
            ach = bytes_b / (us_b * 1e-6) / 1e9
            batch_lines[f"b{b_}"] = {"us_per_step": round(us_b, 3), "us_per_layer": round(us_b / n_layers, 3),
                                     "achieved_gbs": round(ach, 1), "frac": None, "traffic": None}
            tr, _ = engine_traffic(b_)
            batch_lines[f"b{b_}"]["traffic"] = round(tr) if tr else None

    # ---- end to end through the public API with host buffers (N=1 only) ------------------
    # Every step: one H2D copy of the step's 9 activation vectors from pinned host memory, the step's
    # forward (one qp_multi_fwd), one D2H copy of the 9 results into pinned host memory -- captured with
    # the forwards in a CUDA graph per replica (as a serving loop would), timed with events.
    e2e = None
    if not sharded:
        hx = torch.empty(x_elems, dtype=torch.float16).pin_memory()
        hy = torch.empty(y_elems, dtype=torch.float32).pin_memory()
        hx.copy_(bufs[0][0].cpu())
        h2d = hx.numel() * 2
        d2h = hy.numel() * 4
        e2e_graphs = []
        with torch.cuda.stream(stream):
            def e2e_step(rep):
                bufs[rep][0].copy_(hx, non_blocking=True)
                step_fn(rep, stream)
                hy.copy_(bufs[rep][1], non_blocking=True)
            for rep in range(REPLICAS):
                e2e_step(rep)
            stream.synchronize()
            for rep in range(REPLICAS):
                if eager:
                    e2e_graphs.append(None)
                    continue
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    e2e_step(rep)
                e2e_graphs.append(g)

            def run(i):
                g = e2e_graphs[i % REPLICAS]
                if g is None:
                    e2e_step(i % REPLICAS)
                else:
                    g.replay()
            for i in range(args.warmup):
                run(i)
            stream.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(args.steps):
                run(i)
            e1.record(stream)
            e1.synchronize()
        e2e_ms_serial = e0.elapsed_time(e1) / args.steps
        assert torch.isfinite(hy).all(), "non-finite y read back"

        # pipelined, as a serving loop runs it: step i's H2D (its own pinned buffer, copy stream)
        # overlaps step i-1's forwards, and step i's D2H (second copy stream) overlaps step i+1's;
        # every step still moves its inputs in and its results out inside the timed region
        hxs = [hx, torch.empty_like(hx).pin_memory()]
        hys = [hy, torch.empty_like(hy).pin_memory()]
        hxs[1].copy_(hx)
        s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        ev_in = [torch.cuda.Event() for _ in range(REPLICAS)]
        ev_comp = [torch.cuda.Event() for _ in range(REPLICAS)]
        ev_out = [torch.cuda.Event() for _ in range(REPLICAS)]

        def piped(i):
            r = i % REPLICAS
            s_in.wait_event(ev_comp[r])                 # x_r free (step i-2's forwards done)
            with torch.cuda.stream(s_in):
                bufs[r][0].copy_(hxs[r], non_blocking=True)
            ev_in[r].record(s_in)
            stream.wait_event(ev_in[r])
            stream.wait_event(ev_out[r])                # y_r read back (step i-2's D2H done)
            if eager:
                with torch.cuda.stream(stream):
                    step_fn(r, stream)
            else:
                graphs[r].replay()
            ev_comp[r].record(stream)
            s_out.wait_event(ev_comp[r])
            with torch.cuda.stream(s_out):
                hys[r].copy_(bufs[r][1], non_blocking=True)
            ev_out[r].record(s_out)
        with torch.cuda.stream(stream):
            for i in range(args.warmup):
                piped(i)
        torch.cuda.synchronize()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        s_in.wait_event(p0)
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                piped(i)
        s_out.synchronize()
        p1.record(s_out)
        p1.synchronize()
        e2e_ms = p0.elapsed_time(p1) / args.steps
        assert all(torch.isfinite(t).all() for t in hys), "non-finite y read back"
        e2e = {"value": round(step_bytes / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 4),
               "method": "per step: 1 H2D copy of all activations from pinned host memory (copy stream), the "
                         "step's forward (qp_multi_fwd: one engine launch; CUDA graph), 1 D2H copy of all outputs "
                         "into pinned host memory "
                         "(second copy stream); copies of neighbouring steps overlap the forwards; events",
               "serial_value": round(step_bytes / (e2e_ms_serial * 1e-3) / 1e9, 2),
               "serial_ms_per_step": round(e2e_ms_serial, 4)}

    cpu = None
    if rank == 0 and not sharded and not args.no_cpu_baseline:
        nb, dt = oracle_sample(layers, budget_rows=1536)
        cpu = {"value": round(nb / dt / 1e9, 6), "unit": "GB/s", "cores": cpu_cores(), "kind": "oracle",
               "sample": "first 1536 rows of each of the 9 C2 layers: float64 decode + RHT + matvec (batch 1)",
               "seconds": round(dt, 2), **cpu_info()}

    if rank == 0:
        ck = clk.summary()
        peak_b, _ = measured_peaks()
        for k, v in batch_lines.items():
            v["frac"] = round(v["achieved_gbs"] / peak_b, 4)
            v["ceilings"] = ceilings(layers, int(k[1:]), peak_b, ck.get("sm_mhz"))
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f16", "data": "synthetic",
            "config": {"workload": "C2: Llama-3.1-8B (4096x4096, 14336x4096, 4096x14336) x TCQ-2.5 / half-TCQ-3.25 / "
                                   "TCQ-4.0 (L=16), rotation + fused dequant-GEMV per layer on raw fp16 x",
                       "batch": batch, "layers_per_step": n_layers, "us_per_layer": round(ms * 1e3 / n_layers, 3),
                       "parallelism": ((f"row-shard x{world}: engine over each rank's shards with the all-gather "
                                        f"fused into its epilogue (peer stores over NVLink)" if allgather == "p2p" else
                                        f"row-shard x{world}: engine over each rank's shards + one grouped NCCL "
                                        f"all-gather per step") if sharded else "single GPU"),
                       "l2": "inputs larger than L2 (2 replicas, 326 MB per 2 steps, L2 126 MB)",
                       "graph": "CUDA graph per step, PDL between consecutive kernels",
                       "kernels_per_layer": round(launches_per_step / n_layers, 3),
                       "path": ("engine: one persistent qp_multi_fwd launch per step (rotation jobs + all 9 "
                                "GEMVs, device-side ready flags)" if use_engine else
                                "per layer: qp_linear_fwd = rotation kernel + fused GEMV kernel, PDL-chained"),
                       "gemv_us_per_layer": per_layer_us,
                       "independent_steps": indep},
            "roofline": ({"bound": "hbm", "achieved": round(eng["achieved"], 1), "peak": peak, "unit": "GB/s",
                          "frac": round(eng["achieved"] / peak, 4),
                          "traffic": round(eng_traffic) if eng_traffic else None, "traffic_source": eng_traffic_src,
                          "algorithmic_bytes_per_launch": int(eng["bytes"]),
                          "kernel": "qp_engine_kernel (persistent: the 9 layers' rotations + fused dequant-GEMVs in one "
                                    "launch), CUDA graph of back-to-back launches alternating 2 replicas of 163 MB of "
                                    "codes (> L2), events on the launching stream",
                          "peak_kind": peak_kind, "avg_launch_us": round(eng["us"], 3),
                          "ceilings": ceilings(layers, batch, peak, ck.get("sm_mhz")),
                          "batches": batch_lines,
                          "per_layer_path": {"achieved": round(gemv_achieved, 1), "frac": round(gemv_achieved / peak, 4),
                                             "avg_launch_us": round(gemv_avg_ms * 1e3, 3),
                                             "kernel": "qp_gemv_kernel alone per layer (pre-rotated x)"}}
                         if eng else
                         {"bound": "hbm", "achieved": round(gemv_achieved, 1), "peak": peak, "unit": "GB/s",
                          "frac": round(gemv_achieved / peak, 4),
                          "traffic": round(traffic) if traffic else None, "traffic_source": traffic_src,
                          "algorithmic_bytes_per_launch": round(gemv_alg / n_layers),
                          "kernel": "qp_gemv_kernel (fused dequant-GEMV), all 9 layers, CUDA graph of back-to-back "
                                    "launches per layer cycling > 2x L2 of distinct layer copies (codes stream from "
                                    "HBM), events on the launching stream",
                          "peak_kind": peak_kind, "avg_launch_us": round(gemv_avg_ms * 1e3, 3)}),
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches_per_step * args.steps),
            "clocks": ck,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        torch.cuda.synchronize()
        comm.close()
    if sharded:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
