"""One step's kernels, times and DRAM bytes from an ncu --csv launch list
(metrics gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum)
-> profiles/traffic_<cfg>.json, which bench.py reads for roofline.traffic.

    python tools/traffic.py launches.csv <cfg> [--out profiles/traffic_<cfg>.json]

A step starts at a `k_prep` launch (the build's first kernel); the
next-to-last step that ran a traversal kernel is used.  The hot kernel is the step's longest
traversal kernel (k_trav_*); its DRAM bytes per launch are the roofline's
`traffic`, the step's total DRAM bytes go beside it.  ncu's times are
cold-cache and serialised: shares matter, not absolutes.
"""
from __future__ import annotations

import argparse
import csv
import json
from collections import OrderedDict
from pathlib import Path

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
         "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def parse(path):
    lines = Path(path).read_text().splitlines()
    start = [i for i, ln in enumerate(lines) if ln.startswith('"ID"')][0]
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    ki, mi, vi, ii, ui = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID",
                                                "Metric Unit"))
    d = OrderedDict()
    for r in rows[1:]:
        e = d.setdefault(r[ii], {"kernel": r[ki]})
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        e[r[mi]] = v
    return list(d.values())


def short(name: str) -> str:
    base = name.split("(")[0]
    return base.replace("void ", "").replace("rs::", "")


def last_step(launches):
    """The last step (k_prep .. next k_prep) that ran the traversal kernel
    (bench.py's per-segment statistics builds after the timed steps are
    skipped)."""
    starts = [i for i, x in enumerate(launches) if short(x["kernel"]) == "k_prep"]
    bounds = list(zip(starts, starts[1:] + [len(launches)]))
    steps = [launches[a:b] for a, b in bounds]
    with_trav = [st for st in steps if any(short(x["kernel"]).startswith("k_trav") for x in st)]
    if len(with_trav) >= 2:
        return with_trav[-2]  # the last one may be cut short by the capture's end
    return with_trav[-1] if with_trav else (steps[-1] if steps else launches)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("cfg")
    ap.add_argument("--out")
    args = ap.parse_args()
    step = last_step(parse(args.csv))
    rows = []
    for x in step:
        rd, wr = x.get("dram__bytes_read.sum", 0.0), x.get("dram__bytes_write.sum", 0.0)
        rows.append({"kernel": short(x["kernel"]), "us": round(x.get("gpu__time_duration.sum", 0.0), 2),
                     "dram_bytes": int(rd + wr)})
    trav = [r for r in rows if r["kernel"].startswith("k_trav")]
    hot = max(trav, key=lambda r: r["us"]) if trav else max(rows, key=lambda r: r["us"])
    hot_launches = [r for r in rows if r["kernel"] == hot["kernel"]]
    total_us = sum(r["us"] for r in rows)
    out = {
        "kernel": hot["kernel"].split("<")[0],
        "config": args.cfg,
        "dram_bytes_per_launch": int(sum(r["dram_bytes"] for r in hot_launches) / len(hot_launches)),
        "launches_per_step": len(hot_launches),
        "step_dram_bytes": int(sum(r["dram_bytes"] for r in rows)),
        "step_kernel_us": round(total_us, 2),
        "hot_share": round(sum(r["us"] for r in hot_launches) / total_us, 4) if total_us else None,
        "source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                  f"--clock-control none, last complete step of {Path(args.csv).name}",
        "kernels": rows,
    }
    dst = Path(args.out or Path(__file__).resolve().parents[1] / "profiles" / f"traffic_{args.cfg}.json")
    dst.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps({k: v for k, v in out.items() if k != "kernels"}))


if __name__ == "__main__":
    main()
