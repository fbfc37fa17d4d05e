"""Summarise an .ncu-rep (first kernel) into the handful of numbers we track."""
import csv, io, subprocess, sys, json

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "lts__t_sectors_srcunit_tex.sum",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]

def summary(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")][:80]}
        for k in KEYS:
            if k in hdr:
                d[k] = row[hdr.index(k)] + (" " + units[hdr.index(k)] if units[hdr.index(k)] else "")
        out.append(d)
    return out

def stalls(path, top=12):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    r = rows[2]
    st = [(h, float(v)) for h, v in zip(hdr, r) if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith("ratio") is False and v.replace('.','',1).isdigit()]
    st = [(h, v) for h, v in zip(hdr, r) if "warp_latency_issue_stalled" in h]
    res = []
    for h, v in st:
        try: res.append((float(v), h))
        except ValueError: pass
    return sorted(res, reverse=True)[:top]

if __name__ == "__main__":
    for d in summary(sys.argv[1]):
        print(json.dumps(d, indent=1))
    for v, h in stalls(sys.argv[1]):
        print(f"{v:10.3f}  {h}")
