"""Summarise an interleaved A/B run (tools/gpu_round.sh ab): ms/step and the
hot-kernel time per (config, library), best and mean over repetitions."""
import glob
import json
import os
import re
import sys
from collections import defaultdict

d = sys.argv[1]
rows = defaultdict(list)
for f in sorted(glob.glob(os.path.join(d, "ab_*.json"))):
    m = re.match(r"ab_(c\d)_(.+)_(\d+)\.json", os.path.basename(f))
    txt = open(f).read().strip().splitlines()
    if not m or not txt:
        continue
    j = json.loads(txt[-1])
    rows[(m.group(1), m.group(2))].append((j["ms_per_step"], j.get("phase_ms", {}).get("traversal_kernel")))
for (c, lib), v in sorted(rows.items()):
    ms = [x[0] for x in v]
    tk = [x[1] for x in v if x[1] is not None]
    print(f"{c} {lib:>8}  step best {min(ms):.4f} mean {sum(ms)/len(ms):.4f}   "
          f"trav best {min(tk) if tk else float('nan'):.4f}")
