"""Small driver for ncu captures (dev tool): builds one workload and runs a few matvecs per nv.

    python tools/prof_driver.py cfg3s 16 64      # workload, then the nv values
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from h2gen import make_xy, SEED                       # noqa: E402
from h2gen.configs import build_config                # noqa: E402
from paper_2109_05451_b200 import operator_from_h2data, load_library   # noqa: E402

name, nvs = sys.argv[1], [int(v) for v in sys.argv[2:]] or [1]
dtype = os.environ.get("PROF_DTYPE", "f64")
load_library()
h = build_config(name)
op = operator_from_h2data(h, dtype=dtype, nv_max=max(nvs))
tdt = torch.float64 if dtype == "f64" else torch.float32
for nv in nvs:
    X = torch.from_numpy(make_xy(h.perm, nv, SEED)).to("cuda", tdt)
    Y = torch.zeros_like(X)
    for _ in range(3):
        op.matvec(X, Y, 1.0, 0.0)
    torch.cuda.synchronize()
print("done", name, nvs)
