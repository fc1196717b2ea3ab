"""Multi-rank parity on ONE GPU (driver-visible): P ranks emulated in one process by a loopback
group (h2_group_create), so the distributed kernels -- x^ and x-halo packs (k_pack), off-diagonal
coupling from the per-peer receive chunks (k_rows<ACCUM>), the halo-fed dense blocks of
k_leaf_dense and the replicated top tree (k_tree) -- run under `pytest -m gpu` with one device.
The per-call exchange moves the same bytes as the NCCL groups (PAPER.md:445-502,
alg:optimized_dist_mult), by device copies.  Y(P), concatenated in rank order, must match the
oracle's global result within 1e-12 (FP64) / 1e-5 (FP32)."""
import numpy as np
import pytest

import oracle
from h2gen import build_config, make_xy, build_cluster_tree, dual_traversal, random_h2_data
from h2gen.tree import uniform_points
from tests.gpu_util import colmax_rel, with_root_coupling

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2109_05451_b200 import load_library
    load_library()


def _rand(N, m, k, eta, seed):
    tr = build_cluster_tree(uniform_points(N, 2, seed), m)
    st = dual_traversal(tr, eta)
    return random_h2_data(tr, st, [k] * (tr.q + 1), seed)


CASES = {
    "cfg1": lambda: (build_config("cfg1"), 1, "f64"),
    "rand-k25-nv16": lambda: (_rand(6000, 64, 25, 0.9, 5), 16, "f64"),
    "rand-k36-nv3": lambda: (_rand(4000, 32, 36, 0.9, 6), 3, "f64"),
    "rand-k25-nv20-chunks": lambda: (_rand(5000, 64, 25, 0.9, 8), 20, "f64"),
    "rand-k64-nv64": lambda: (_rand(4000, 64, 64, 1.1, 10), 64, "f64"),
    "rand-k16-fp32-nv5": lambda: (_rand(4000, 32, 16, 0.9, 9), 5, "f32"),
    # tcgen05 FP32 coupling with the x^ tensor map (k = 64, nv % 8 == 0) and the off-diagonal
    # blocks from the received x^ (per-vector bulk copies)
    "rand-k64-fp32-nv16": lambda: (_rand(4000, 64, 64, 1.1, 13), 16, "f32"),
    "top-tree-eta3": lambda: (_rand(5000, 32, 16, 3.0, 7), 2, "f64"),
    "top-tree-root-block": lambda: (with_root_coupling(_rand(3000, 32, 12, 0.9, 12)), 4, "f64"),
}


def run_group(h, P, nv, dt):
    import torch
    from paper_2109_05451_b200 import group_from_h2data
    hh = h.astype(np.float32) if dt == "f32" else h
    grp, rows = group_from_h2data(hh, P, dtype=dt, nv_max=nv)
    npdt = np.float64 if dt == "f64" else np.float32
    X = make_xy(h.perm, nv, 11, -1.0, 1.0).astype(npdt)
    Y0 = make_xy(h.perm, nv, 12, -1.0, 1.0, stream=1).astype(npdt)
    Xs = [torch.from_numpy(np.ascontiguousarray(X[:, a:b])).cuda() for a, b in rows]
    outs = []
    for rep in range(2):                         # repeated calls reuse the buffers
        Ys = [torch.from_numpy(np.ascontiguousarray(Y0[:, a:b])).cuda() for a, b in rows]
        grp.matvec(Xs, Ys, 0.75, -0.5)
        torch.cuda.synchronize()
        outs.append(np.concatenate([y.cpu().numpy() for y in Ys], axis=1).astype(np.float64))
    counts = [grp.plan_counts(o) for o in range(P)]
    grp.close()
    ref = oracle.matvec(hh.astype(np.float64) if dt == "f32" else h, X.astype(np.float64), 0.75, -0.5,
                        Y0.astype(np.float64))
    return outs, ref, counts


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("name", sorted(CASES))
def test_loopback_parity(name, P):
    h, nv, dt = CASES[name]()
    outs, ref, counts = run_group(h, P, nv, dt)
    tol = 1e-12 if dt == "f64" else 1e-5
    for out in outs:
        assert colmax_rel(out, ref) <= tol
    assert np.array_equal(outs[0], outs[1])
    off = sum(c["offdiag_S"] for c in counts)
    assert off > 0, "the case must exercise the off-diagonal exchange"
    if name.startswith("top-tree"):
        root = sum(c["root_S"] for c in counts)
        if name == "top-tree-root-block" or P == 4:
            assert root > 0, "the top-tree case must hold root-branch couplings"


def test_root_block_single_rank():
    """The root-coupling structure on one rank (C = 0: the root is an ordinary level)."""
    import torch
    from paper_2109_05451_b200 import operator_from_h2data
    h = with_root_coupling(_rand(3000, 32, 12, 0.9, 12))
    op = operator_from_h2data(h, nv_max=4)
    X = make_xy(h.perm, 4, 11, -1.0, 1.0)
    Y0 = make_xy(h.perm, 4, 12, -1.0, 1.0, stream=1)
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y0.copy()).cuda()
    op.matvec(Xd, Yd, 0.75, -0.5)
    torch.cuda.synchronize()
    op.close()
    assert colmax_rel(Yd.cpu().numpy(), oracle.matvec(h, X, 0.75, -0.5, Y0)) <= 1e-12
