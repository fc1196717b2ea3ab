"""Time h2_orthogonalize and h2_reweigh (NEXT-3 steps 1-2) on full-size workloads (dev / evidence tool).

    python tools/bench_orth.py cfg2 cfg5        # FP64; prints one JSON line per workload
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from h2gen.configs import build_config
from paper_2109_05451_b200 import operator_from_h2data, load_library

load_library()
for name in sys.argv[1:] or ["cfg2"]:
    h = build_config(name)
    q, m, k = h.q, h.m, h.ranks
    # flops: Householder QR + explicit Q of an r x c matrix ~ 4 r c^2 - 4 c^3 / 3; stack GEMMs
    # 2 (2 k^l k^l k^{l-1}) per parent; projection 4 k^3 per coupling block (both trees for QR)
    qr = lambda r, c: 4.0 * r * c * c - 4.0 * c ** 3 / 3.0
    fl = 2 * (1 << q) * qr(m, k[q])
    for l in range(1, q + 1):
        np_ = 1 << (l - 1)
        fl += 2 * np_ * (qr(2 * k[l], k[l - 1]) + 2 * 2.0 * k[l] * k[l] * k[l - 1])
    fl += sum(4.0 * s.shape[0] * k[l] ** 3 for l, s in enumerate(h.S))
    bytes_ = 8 * 2 * (h.U_leaf.size + h.V_leaf.size + sum(e.size for e in h.E[1:]) * 2 + sum(s.size for s in h.S))
    res, rw = [], []
    nR = sum((1 << l) * k[l] ** 2 for l in range(q + 1))
    for rep in range(3):
        op = operator_from_h2data(h, nv_max=1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op.orthogonalize()
        res.append(time.perf_counter() - t0)
        Rd = torch.empty(nR, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op.reweigh(Rd)
        rw.append(time.perf_counter() - t0)
        del Rd
        op.close()
    t = min(res)
    print(json.dumps({"workload": name, "ms": t * 1e3, "ms_all": [r * 1e3 for r in res], "gflops": fl / t / 1e9,
                      "gb_moved_min": bytes_ / 1e9, "gbs": bytes_ / t / 1e9,
                      "reweigh_ms": min(rw) * 1e3, "reweigh_ms_all": [r * 1e3 for r in rw], "leaves": 1 << q, "m": m, "k": k[q]}))
