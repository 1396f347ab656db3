"""Write profiles/traffic.json: DRAM bytes (read + write) per launch for each
pipeline stage, from one `ncu --set full` capture of bench.py. bench.py puts the
dominant stage's value into its roofline line as `traffic`.

    python tools/ncu_traffic.py gpurun_out/prof_rXX.ncu-rep
"""
import csv
import json
import pathlib
import subprocess
import sys

STAGE = {"k_blur_stencil": "antialias", "k_blur_runs": "antialias", "k_lanczos_smem": "warp",
         "k_lanczos_sep": "warp_sep", "k_warp": "warp", "k_pyramid": "pyramid", "k_fast_nms": "fast_nms",
         "k_measures": "measures", "k_select": "select", "k_orient": "select", "k_describe": "describe",
         "k_match_jobs": "match", "k_match_umma": "match", "k_match_partial": "hamming"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(raw))
h, units = rows[0], rows[1]
ki = h.index("Kernel Name")
out = {}
for x in rows[2:]:
    name = x[ki].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1].strip()
    st = STAGE.get(name)
    if not st:
        continue
    b = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(m)
        b += float(x[i]) * UNIT.get(units[i], 1)
    dur = float(x[h.index("gpu__time_duration.sum")].replace(",", ""))
    out.setdefault(st, []).append((dur, b))
# per launch: the mean over a stage's launches, except for the stages that also
# have a short once-per-call zero-fill launch of the same kernel (k_pyramid<1>,
# the zpass-1 k_lanczos_smem): there the main (longest) launch
res = {k: (max(v)[1] if k in ("warp", "pyramid") else sum(b for _, b in v) / len(v)) for k, v in out.items()}
res["_source"] = rep
path = pathlib.Path(__file__).resolve().parents[1] / "profiles" / "traffic.json"
path.write_text(json.dumps(res, indent=1) + "\n")
print(json.dumps(res, indent=1))
