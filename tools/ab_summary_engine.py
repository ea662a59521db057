"""Summarise scripts/ab_engine_vs_head.sh output: us per launch per (arm, batch, set), runs side by side."""
import json
import sys

cur, res = None, {}
for line in open(sys.argv[1]):
    line = line.strip()
    if line.split(" ")[0] in ("old", "new", "base", "mulhi", "v3", "cur", "head", "cur_rp", "np", "rp", "va", "vb"):
        cur = line
    elif line.startswith("{"):
        d = json.loads(line)
        res.setdefault((d["set"], cur.split()[1], cur.split()[0]), []).append(d["us_per_launch"])
for (st, b, arm), v in sorted(res.items()):
    print(f"{st:10s} {b} {arm:4s} " + " ".join(f"{x:7.2f}" for x in v))
