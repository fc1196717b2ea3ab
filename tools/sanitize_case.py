"""Small cases for compute-sanitizer (one tool per gpurun call): cfg1 and a ragged random
structure, SIMT (nv=1,3) and DMMA (nv=8) engines, eager + graph calls, parity checked."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from h2gen import build_config, make_xy
from tests.gpu_util import random_case, gpu_matvec, colmax_rel
from paper_2109_05451_b200 import operator_from_h2data
cases = [("cfg1", build_config("cfg1")), ("ragged", random_case(900, 32, lambda l: 12 + (l % 3) * 7, 4))]
worst = 0.0
for name, h in cases:
    for nv in (1, 3, 8):
        op = operator_from_h2data(h, nv_max=nv)
        X = make_xy(h.perm, nv, 1, -1.0, 1.0)
        Y0 = make_xy(h.perm, nv, 2, -1.0, 1.0, stream=1)
        ref = oracle.matvec(h, X, 0.5, 0.25, Y0)
        for rep in range(3):
            out = gpu_matvec(op, X, 0.5, 0.25, Y0)
            worst = max(worst, colmax_rel(out, ref))
        op.close()
        print(name, nv, "ok", flush=True)
print("worst rel err", worst)
sys.exit(0 if worst <= 1e-12 else 1)
