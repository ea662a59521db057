"""Summarise scripts/ab3.sh output: minimum us/launch per (variant, config) and the per-variant sum."""
import collections
import re
import sys

best = collections.defaultdict(dict)
for line in open(sys.argv[1]):
    if "|" not in line or "us/launch" not in line:
        continue
    lib, rest = [x.strip() for x in line.split("|", 1)]
    cfg = rest.split(" (graph")[0]
    us = float(re.search(r"([0-9.]+) us/launch", rest).group(1))
    best[cfg][lib] = min(us, best[cfg].get(lib, 1e9))
libs = sorted({lib for c in best.values() for lib in c})
print("config".ljust(40) + "".join(lib[:22].rjust(24) for lib in libs))
tot = collections.Counter()
for cfg, d in best.items():
    print(cfg.ljust(40) + "".join(f"{d.get(lib, float('nan')):24.2f}" for lib in libs))
    for lib in libs:
        tot[lib] += d.get(lib, 0)
print("sum".ljust(40) + "".join(f"{tot[lib]:24.2f}" for lib in libs))
