"""Symmetric storage (h2_desc.flags = H2_SYMMETRIC): only the blocks
(t, s), t <= s, are stored and the others applied as transposes.  The oracle runs the FULL
(unsymmetric-storage) operator; the GPU result must match it within 1e-12 (FP64) / 1e-5 (FP32),
and equal the general-storage GPU result to the same tolerance."""
import dataclasses

import numpy as np
import pytest

import oracle
from h2gen import build_config, make_xy
from tests.gpu_util import colmax_rel, random_case, gpu_matvec

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2109_05451_b200 import load_library
    load_library()


def symmetrize(h):
    """Random H² data made symmetric: U = V, E = F, S_st = S_ts^T, D_st = D_ts^T (D_tt symmetric)."""
    S = [s.copy() for s in h.S]
    for l in range(h.q + 1):
        rp, col = h.S_rowptr[l], h.S_col[l]
        pos = {}
        for t in range(rp.size - 1):
            for b in range(rp[t], rp[t + 1]):
                pos[(t, int(col[b]))] = b
        for (t, s_), b in pos.items():
            if s_ < t:
                S[l][b] = S[l][pos[(s_, t)]].T          # stored [blk][col][row]: transpose = swap axes
    D = h.D.copy()
    rp, col = h.D_rowptr, h.D_col
    pos = {(t, int(col[b])): b for t in range(rp.size - 1) for b in range(rp[t], rp[t + 1])}
    for (t, s_), b in pos.items():
        if s_ < t:
            D[b] = D[pos[(s_, t)]].T
        elif s_ == t:
            D[b] = 0.5 * (D[b] + D[b].T)
    return dataclasses.replace(h, V_leaf=h.U_leaf, F=h.E, S=S, D=D)


def run(h, nv=1, dtype="f64", alpha=-0.7, beta=0.3, seed=3):
    from paper_2109_05451_b200 import operator_from_h2data
    X = make_xy(h.perm, nv, seed, -1.0, 1.0)
    Y0 = make_xy(h.perm, nv, seed + 1, -1.0, 1.0, stream=1)
    hh = h if dtype == "f64" else h.astype(np.float32)
    if dtype == "f32":
        X, Y0 = X.astype(np.float32).astype(np.float64), Y0.astype(np.float32).astype(np.float64)
    op = operator_from_h2data(hh, nv_max=nv, dtype=dtype, symmetric=True)
    out = gpu_matvec(op, X, alpha, beta, Y0, dtype)
    st = op.stats(1)
    op.close()
    ref = oracle.matvec(hh.astype(np.float64) if dtype == "f32" else h, X, alpha, beta, Y0)
    return out, ref, st


@pytest.mark.parametrize("name", ["cfg1", "cfg1grid"])
def test_symmetric_kernel_configs(name):
    out, ref, _ = run(build_config(name))
    assert colmax_rel(out, ref) <= 1e-12


@pytest.mark.parametrize("N,m,k,seed", [(3000, 32, 16, 1), (4000, 64, 25, 2), (2500, 48, 36, 3), (3000, 64, 64, 4)])
def test_symmetric_random(N, m, k, seed):
    h = symmetrize(random_case(N, m, lambda l: k, seed))
    out, ref, _ = run(h, beta=0.0)
    assert colmax_rel(out, ref) <= 1e-12
    out, ref, _ = run(h, alpha=1.5, beta=-2.0)
    assert colmax_rel(out, ref) <= 1e-12


def test_symmetric_fp32():
    h = symmetrize(random_case(3000, 64, lambda l: 25, 9))
    out, ref, _ = run(h, dtype="f32")
    assert colmax_rel(out, ref) <= 1e-5


def test_symmetric_stores_about_half():
    from paper_2109_05451_b200 import operator_from_h2data
    h = build_config("cfg1")
    full = operator_from_h2data(h, nv_max=1)
    half = operator_from_h2data(h, nv_max=1, symmetric=True)
    f, s = full.stats(1), half.stats(1)
    full.close()
    half.close()
    assert f["flops"] == s["flops"]                      # same operator, same flop model
    assert s["bytes"] < 0.75 * f["bytes"]


def test_symmetric_rejects_nv_max_above_one():
    from paper_2109_05451_b200 import operator_from_h2data, H2Error
    with pytest.raises(H2Error):
        operator_from_h2data(build_config("cfg1"), nv_max=2, symmetric=True)


@pytest.mark.slow
def test_symmetric_cfg2_full_size_sampled():
    h = build_config("cfg2")
    from paper_2109_05451_b200 import operator_from_h2data
    X = make_xy(h.perm, 1, 3, 0.0, 1.0)
    op = operator_from_h2data(h, nv_max=1, symmetric=True)
    out = gpu_matvec(op, X, 1.0, 0.0, np.zeros_like(X))
    op.close()
    mask = np.zeros(1 << h.q, dtype=bool)
    mask[np.random.default_rng(2).choice(mask.size, mask.size // 50, replace=False)] = True
    mask[[0, -1]] = True
    ref = oracle.matvec(h, X, 1.0, 0.0, None, leaf_mask=mask)
    rows = np.concatenate([np.arange(h.leaf_ptr[i], h.leaf_ptr[i + 1]) for i in np.flatnonzero(mask)])
    assert colmax_rel(out[:, rows], ref[:, rows]) <= 1e-12
