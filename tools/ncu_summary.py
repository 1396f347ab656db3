"""Summarise an `ncu --set full` report into a markdown table under profiles/.

    python tools/ncu_summary.py gpurun_out/prof_rXX.ncu-rep profiles/rXX_ncu.md "title"
"""
import csv
import subprocess
import sys

rep, out, title = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
r = list(csv.reader(raw))
h, units = r[0], r[1]
ki = h.index("Kernel Name")
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def dur_ms(x):
    i = h.index("gpu__time_duration.sum")
    v = float(x[i].replace(",", ""))
    return v * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(units[i], 1.0)


def g(x, n):
    return x[h.index(n)] if n in h else ""


def gb(x, n):
    i = h.index(n)
    return float(x[i]) * UNIT.get(units[i], 1) / 1e9


PIPES = ["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
         "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
         "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
         "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
         "l1tex__throughput.avg.pct_of_peak_sustained_active",
         "lts__throughput.avg.pct_of_peak_sustained_elapsed"]


def pct(x, n):
    try:
        return float(g(x, n))
    except ValueError:
        return float("nan")


stall = [i for i, n in enumerate(h) if n.startswith("smsp__average_warps_issue_stalled_")
         and n.endswith("_per_issue_active.ratio")]
lines = [f"# {title}", "", f"source: `{rep}` (ncu --set full --clock-control none, one B200)", "",
         "Pipe columns: % of peak while the SM is active (FMA / ALU / XU (MUFU, conversions, POPC) / "
         "LSU issue), L1 = l1tex throughput (shared + global wavefronts), L2 = lts throughput.", "",
         "| kernel | ms | warp-inst (M) | issue % | occupancy % | regs | FMA % | ALU % | XU % | LSU % | L1 % "
         "| L2 % | DRAM rd GB | DRAM wr GB | top stalls |",
         "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
for x in r[2:]:
    st = []
    for i in stall:
        try:
            st.append((float(x[i]), h[i][len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
    st.sort(reverse=True)
    name = x[ki].split("(")[0].replace("void ", "")
    lines.append(
        f"| {name} | {dur_ms(x):.3f} | "
        f"{float(g(x, 'smsp__inst_executed.sum')) / 1e6:.0f} | "
        f"{float(g(x, 'sm__inst_issued.avg.pct_of_peak_sustained_active')):.0f} | "
        f"{float(g(x, 'sm__warps_active.avg.pct_of_peak_sustained_active')):.0f} | "
        f"{g(x, 'launch__registers_per_thread')} | "
        + " | ".join(f"{pct(x, m):.0f}" for m in PIPES) + " | "
        f"{gb(x, 'dram__bytes_read.sum'):.3f} | {gb(x, 'dram__bytes_write.sum'):.3f} | "
        + ", ".join(f"{n} {v:.1f}" for v, n in st[:4]) + " |")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
