"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into a
markdown table (per kernel: launches, mean us, share of this repo's kernel time).

usage: python tools/launch_list.py gpurun_out/launches.csv profiles/rXX_launches.md "title"
"""
import collections
import csv
import sys


def main():
    src, out, title = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    t = collections.OrderedDict()
    for r in rows[1:]:
        if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0]
        v = float(r[iv].replace(",", ""))
        v = v / 1e3 if r[iu] == "ns" else (v * 1e3 if r[iu] == "ms" else v)  # -> us
        t.setdefault(name, []).append(v)
    mine = {k: v for k, v in t.items() if "xa::" in k or "k_" in k}
    tot = sum(sum(v) for v in mine.values()) or 1.0
    lines = [f"# {title}", "",
             "Cold-cache, serialised per-launch times (ncu); compare shares, not absolutes.", "",
             "| kernel | launches | mean us | share of xa time |", "|---|---|---|---|"]
    for k, v in mine.items():
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / tot:.1f}% |")
    other = {k: v for k, v in t.items() if k not in mine}
    if other:
        lines += ["", "Other kernels in the process (torch: L2 flush, input setup): "
                  + ", ".join(f"{k} x{len(v)}" for k, v in other.items())]
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
