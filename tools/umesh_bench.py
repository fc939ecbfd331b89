"""Element-list operator sweep alone (bench.umesh_sweep), one JSON line; optional argv:
`dim n` runs a single mesh (for ncu captures)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1511_08463_b200 as pf  # noqa: E402

if len(sys.argv) == 3:
    bench.UMESH_SWEEP = ((int(sys.argv[1]), int(sys.argv[2])),)
peak, kind = bench.peaks()
print(json.dumps({"peak_GB_s": peak, "peak_kind": kind,
                  "operator_sweep_unstructured": bench.umesh_sweep(pf, torch, peak, reps=10)}))
