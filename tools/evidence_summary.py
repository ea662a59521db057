"""Summaries of a GPU evidence run (scripts/round_evidence_r2.sh): the ncu launch list of the bench
step and the ncu --set full metrics of the engine kernel at batch 1 / 8, as markdown.

    python tools/evidence_summary.py ev7 profiles/r2/v7
"""
import collections
import csv
import os
import re
import subprocess
import sys


def launches(tag, out_dir):
    rows = list(csv.reader(open(f"gpurun_out/{tag}_launches.csv")))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ix = {h: i for i, h in enumerate(hdr)}
    seq = []
    for r in data:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        us = v / 1000 if unit in ("nsecond", "ns") else (v * 1000 if unit in ("msecond", "ms") else v)
        seq.append((r[ix["Kernel Name"]], us))
    out = [f"# ncu launch list of the bench step ({tag})", "",
           "`QP_BENCH_EAGER=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py "
           "--steps 3 --warmup 3` (eager replay: ncu cannot profile inside CUDA graphs). The first launches are the "
           "bench steps: ONE `qp_engine_kernel` per step (the 9 layers' rotations + fused dequant-GEMVs); later "
           "launches belong to bench.py's per-layer comparison section. ncu serialises launches with cold caches, "
           "so absolute times are above the graph-timed ones; the engine kernel is 100% of the step.", "",
           "| # | kernel | us |", "|---|---|---|"]
    out += [f"| {i} | `{n[:70]}` | {us:.2f} |" for i, (n, us) in enumerate(seq[:12])]
    agg = collections.OrderedDict()
    for n, us in seq:
        agg.setdefault(n, []).append(us)
    out += ["", "All captured launches:", "", "| kernel | n | avg us |", "|---|---|---|"]
    out += [f"| `{n[:80]}` | {len(v)} | {sum(v) / len(v):.2f} |" for n, v in agg.items()]
    open(os.path.join(out_dir, "launches_summary.md"), "w").write("\n".join(out) + "\n")


WANT = [("gpc__cycles_elapsed.max", "Elapsed cycles"), ("gpu__time_duration.sum", "Duration (us)"),
        ("sm__cycles_active.avg", "SM active cycles"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "Issue slots busy %"),
        ("smsp__average_warp_latency_per_inst_issued.ratio", "Warp cycles per issued instruction"),
        ("dram__bytes_read.sum", "DRAM MB read"), ("dram__bytes_write.sum", "DRAM MB written"),
        ("smsp__inst_executed.sum", "Warp instructions executed"), ("launch__registers_per_thread", "Registers / thread"),
        ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"), ("lts__t_sector_hit_rate.pct", "L2 hit rate %")]


def ncu_full(tag, out_dir):
    vals, stalls = {}, {}
    for b, rep in (("1", f"{tag}_prof_engine"), ("8", f"{tag}_prof_engine_b8")):
        txt = subprocess.run(["ncu", "-i", f"gpurun_out/{rep}.ncu-rep", "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(txt.splitlines()))
        hdr, r = rows[0], rows[2]
        ix = {h: i for i, h in enumerate(hdr)}
        vals[b] = {k: r[ix[k]] for k, _ in WANT}
        st = [(float(r[ix[h]] or 0), re.sub(r"smsp__average_warps?_issue_stalled_|_per_issue_active.ratio", "", h))
              for h in hdr if "issue_stalled" in h and h.endswith("per_issue_active.ratio") and "not_issued" not in h]
        stalls[b] = ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:8])
    out = [f"# ncu --set full: the persistent engine kernel, C2 step ({tag})", "",
           "`ncu --set full --clock-control none --import-source on -k regex:qp_engine_kernel -s 4 -c 1 python "
           "tools/engine_ab.py --sets c2 --eager --iters 1 [--batch 8]` on one B200: `qp_engine_kernel<0,16,9,32,5,8,1>` "
           "(TCQ tb = 9, c in [5, 8]), grid 148 x 512, the 9 C2 layers (rotation jobs + fused dequant-GEMVs) in one "
           "launch. ncu replays with cold caches and its own clocks: absolute times are above the graph-timed ones.", "",
           "| metric | batch 1 | batch 8 |", "|---|---|---|"]
    out += [f"| {name} (`{k}`) | {vals['1'][k]} | {vals['8'][k]} |" for k, name in WANT]
    out += ["", "Stall reasons, cycles per issued instruction:", "", f"* batch 1: {stalls['1']}",
            f"* batch 8: {stalls['8']}"]
    open(os.path.join(out_dir, "ncu_engine_full.md"), "w").write("\n".join(out) + "\n")


if __name__ == "__main__":
    tag, out_dir = sys.argv[1], sys.argv[2]
    os.makedirs(out_dir, exist_ok=True)
    launches(tag, out_dir)
    ncu_full(tag, out_dir)
