"""Per-source-line hot spots of one kernel in an ncu report (needs -lineinfo and
--import-source on): instructions executed and stall samples per CUDA line.

    python tools/ncu_lines_hot.py REPORT.ncu-rep KERNEL_REGEX [top=25]
"""
import csv
import io
import os
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                          "--launch-skip", os.environ.get("SKIP", "0"), "--launch-count", "1", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows, fname, hdr = [], "", None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0].isdigit():
            rows.append((fname, r))
    if not hdr:
        print("no source rows")
        return
    ii = hdr.index("Instructions Executed")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    tot_i = sum(float(r[ii] or 0) for _, r in rows) or 1.0
    tot_s = sum(float(r[si] or 0) for _, r in rows) or 1.0
    rows.sort(key=lambda fr: -float(fr[1][ii] or 0))
    print(f"{'file:line':28s} {'inst%':>6s} {'stall%':>6s}  source")
    for f, r in rows[:top]:
        print(f"{f + ':' + r[0]:28s} {100 * float(r[ii] or 0) / tot_i:6.1f} {100 * float(r[si] or 0) / tot_s:6.1f}  "
              f"{r[1].strip()[:90]}")


if __name__ == "__main__":
    main()
