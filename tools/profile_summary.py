"""Turn a gpurun_out/<tag>/ capture into the tracked profiles/ summary.

    python tools/profile_summary.py gpurun_out/<tag> profiles/<name>

Writes <name>/launches_step.md (one full step of the ncu launch list,
gpu__time_duration per kernel and its share of the step) and
<name>/kernels.json (per-kernel ncu --set full metrics: duration, DRAM bytes,
L1/L2 hit rates, issue activity, achieved occupancy, registers)."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def launches(src: Path):
    lines = (src / "launches.csv").read_text().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    ks = [(r[ki], float(r[vi]) / 1e3) for r in rows[1:] if len(r) > vi]
    return [k for k in ks if "at::" not in k[0]]


def one_step(ks):
    # the last step: from the last k_prep to the end
    last = max(i for i, k in enumerate(ks) if "k_prep" in k[0])
    return ks[last:]


def full(src: Path):
    rep = src / "full.ncu-rep"
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                d[k] = r[hdr.index(k)] + (" " + units[hdr.index(k)] if units[hdr.index(k)] else "")
        out.append(d)
    return out


def main():
    src, dst = Path(sys.argv[1]), Path(sys.argv[2])
    dst.mkdir(parents=True, exist_ok=True)
    step = one_step(launches(src))
    tot = sum(t for _, t in step)
    md = ["| kernel | us | share |", "|---|---:|---:|"]
    for name, t in step:
        md.append(f"| `{name.split('(')[0]}` | {t:.2f} | {100 * t / tot:.1f}% |")
    md.append(f"| **sum of kernels, one step** | **{tot:.2f}** | 100% |")
    (dst / "launches_step.md").write_text(
        "ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised;"
        " compare shares, not absolutes)\n\n" + "\n".join(md) + "\n")
    if (src / "full.ncu-rep").exists():
        (dst / "kernels.json").write_text(json.dumps(full(src), indent=1))
    print("\n".join(md))


if __name__ == "__main__":
    main()
