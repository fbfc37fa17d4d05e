"""Per-source-line instruction counts and stall samples from an .ncu-rep.

    python tools/ncu_lines.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    by = sys.argv[4] if len(sys.argv) > 4 else "stall"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = []
    seen = set()
    fname = None
    hdr = None
    for r in csv.reader(io.StringIO(raw)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "" or r[0] == "Function Name":
            continue
        try:
            samp = int(r[4]); inst = int(r[7])
        except (ValueError, IndexError):
            continue
        key = (fname, r[0])
        if key in seen:
            continue
        seen.add(key)
        rows.append((inst, samp, f"{fname}:{r[0]}", r[1][:90]))
    tot_i = sum(x[0] for x in rows) or 1
    tot_s = sum(x[1] for x in rows) or 1
    print(f"total warp-inst {tot_i}  samples {tot_s}")
    for inst, samp, loc, src in sorted(rows, key=lambda x: -x[1] if by == "stall" else -x[0])[:top]:
        print(f"{100*inst/tot_i:5.1f}% inst {100*samp/tot_s:5.1f}% stall  {loc:22s} {src}")


if __name__ == "__main__":
    main()
