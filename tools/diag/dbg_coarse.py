import sys, os
sys.path.insert(0, ".")
import numpy as np
import paper_2503_03479_b200 as xa
from paper_2503_03479_b200 import synth
a, b = synth.config1(seed=3)
g = xa.build_param_grid(xa.GridConfig(n=3))
try:
    r = xa.coarse_search(a, b, g, 500, 0.8, warp_mode="lanczos")
    print("ok", [c for _, c in r.per_entry_counts][:6])
except Exception as e:
    print("ERR", e)
