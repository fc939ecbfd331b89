"""The element-list operator sweep of bench.py alone (jittered 1024^2..4096^2, 64^3..128^3)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1511_08463_b200 as pf

peak, _ = bench.peaks()
for r in bench.umesh_sweep(pf, torch, peak):
    print(json.dumps({k: (round(v, 5) if isinstance(v, float) else v) for k, v in r.items()
                      if k in ("op", "mesh", "median_s", "GB_s", "frac")}))
