"""Localize a parity failure: dense-only / low-rank-only variants across nv (debug tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from h2gen import make_xy
from tests.gpu_util import random_case, gpu_matvec, colmax_rel
from paper_2109_05451_b200 import operator_from_h2data
h = random_case(3000, 64, lambda l: 25, 3)
for variant in ("full", "dense_only", "lowrank_only"):
    hv = random_case(3000, 64, lambda l: 25, 3)
    if variant == "dense_only":
        hv.S = [np.zeros_like(s) for s in hv.S]
    if variant == "lowrank_only":
        hv.D = np.zeros_like(hv.D)
    for nv in (1, 4, 8, 16, 17):
        op = operator_from_h2data(hv, nv_max=nv)
        X = make_xy(hv.perm, nv, 3, -1.0, 1.0)
        Y0 = make_xy(hv.perm, nv, 3, -1.0, 1.0, stream=1)
        ref = oracle.matvec(hv, X, 1.3, -0.4, Y0)
        out = gpu_matvec(op, X, 1.3, -0.4, Y0)
        errs = [np.linalg.norm(out[i] - ref[i]) / np.linalg.norm(ref[i]) for i in range(nv)]
        print(variant, nv, "max col err %.2e" % max(errs), "worst col", int(np.argmax(errs)), flush=True)
        op.close()
