"""Per-source-line instruction and stall-sample totals for one kernel of an
ncu report (needs -lineinfo + --import-source on).

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [top_n]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "-c", "1", "--page", "source", "--csv",
                          "--print-source=cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, agg = "", None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0] or len(r) < len(hdr):
            continue
        ie = hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            agg.append((int(r[ie] or 0), int(r[ss] or 0), f"{fname}:{r[0]}", r[1].strip()[:90]))
        except ValueError:
            pass
    tot_i = sum(a[0] for a in agg) or 1
    tot_s = sum(a[1] for a in agg) or 1
    print(f"total instructions {tot_i/1e6:.1f} M, stall samples {tot_s}")
    for a in sorted(agg, key=lambda a: -a[0])[:top]:
        print(f"{100*a[0]/tot_i:5.1f}% inst {100*a[1]/tot_s:5.1f}% stall  {a[2]:<20} {a[3]}")


if __name__ == "__main__":
    main()
