"""Parity of the CUDA path (through the C ABI) with the CPU oracle, element by element on the
same seeded inputs.  Tolerances (north_star): relative 2-norm <= 1e-12 per
column in FP64; <= 1e-5 in FP32 against the FP64 oracle run on the FP32-rounded inputs."""
import numpy as np
import pytest

import oracle
from h2gen import build_config, make_xy
from tests.gpu_util import colmax_rel, random_case, gpu_matvec

pytestmark = pytest.mark.gpu

TOL64, TOL32 = 1e-12, 1e-5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2109_05451_b200 import load_library
    load_library()


def _op(h, **kw):
    from paper_2109_05451_b200 import operator_from_h2data
    return operator_from_h2data(h, **kw)


def test_cfg1_parity():
    h = build_config("cfg1")
    op = _op(h, nv_max=1)
    X = make_xy(h.perm, 1, 1, -1.0, 1.0)
    Y0 = make_xy(h.perm, 1, 2, -1.0, 1.0, stream=1)
    ref = oracle.matvec(h, X, -0.7, 0.3, Y0)
    out = gpu_matvec(op, X, -0.7, 0.3, Y0)
    assert colmax_rel(out, ref) <= TOL64


@pytest.mark.parametrize("N,m,kfn,nv,seed", [
    (700, 16, lambda l: 5 + (l * 3) % 9, 1, 1),           # ragged leaves, varying small ranks
    (2000, 32, lambda l: 16, 3, 2),
    (3000, 64, lambda l: 25, 17, 3),                      # k = 25, nv = 17 (two vector chunks)
    (3000, 64, lambda l: 36, 16, 4),
    (2500, 64, lambda l: 64, 2, 5),                       # k = 64 (two rows per lane)
    (1500, 32, lambda l: 40 if l % 2 else 20, 64, 6),     # k alternating across 32, nv = 64
    (1000, 64, lambda l: 33, 5, 7),
])
def test_random_structures(N, m, kfn, nv, seed):
    h = random_case(N, m, kfn, seed)
    op = _op(h, nv_max=nv)
    X = make_xy(h.perm, nv, seed, -1.0, 1.0)
    Y0 = make_xy(h.perm, nv, seed, -1.0, 1.0, stream=1)
    ref = oracle.matvec(h, X, 1.3, -0.4, Y0)
    out = gpu_matvec(op, X, 1.3, -0.4, Y0)
    assert colmax_rel(out, ref) <= TOL64


def test_beta_zero_nan_and_alpha_zero():
    h = random_case(900, 32, lambda l: 12, 11)
    op = _op(h, nv_max=2)
    X = make_xy(h.perm, 2, 1, -1.0, 1.0)
    Ynan = np.full((2, h.N), np.nan)
    out = gpu_matvec(op, X, 0.9, 0.0, Ynan)
    assert np.all(np.isfinite(out))
    assert colmax_rel(out, oracle.matvec(h, X, 0.9)) <= TOL64
    Y0 = make_xy(h.perm, 2, 3, stream=1)
    out = gpu_matvec(op, X, 0.0, 0.5, Y0)
    assert np.array_equal(out, 0.5 * Y0)


def test_nv_smaller_than_nv_max_and_repeat_calls():
    h = random_case(1200, 32, lambda l: 16, 12)
    op = _op(h, nv_max=16)
    for nv in (1, 5, 16):
        X = make_xy(h.perm, nv, nv, -1.0, 1.0)
        ref = oracle.matvec(h, X)
        for _ in range(2):
            out = gpu_matvec(op, X, 1.0, 0.0, np.zeros_like(X))
            assert colmax_rel(out, ref) <= TOL64


def test_device_adopted_equals_host_copied():
    h = random_case(1500, 32, lambda l: 16, 13)
    X = make_xy(h.perm, 4, 1, -1.0, 1.0)
    a = gpu_matvec(_op(h, nv_max=4), X, 1.0, 0.0, np.zeros_like(X))
    b = gpu_matvec(_op(h, nv_max=4, device=True), X, 1.0, 0.0, np.zeros_like(X))
    assert np.array_equal(a, b)


def test_fp32_path():
    h = random_case(2000, 64, lambda l: 25, 14)
    h32 = h.astype(np.float32)
    op = _op(h32, nv_max=16, dtype="f32")
    X = make_xy(h.perm, 16, 1, -1.0, 1.0).astype(np.float32)
    Y0 = make_xy(h.perm, 16, 2, -1.0, 1.0, stream=1).astype(np.float32)
    ref = oracle.matvec(h32.astype(np.float64), X.astype(np.float64), 1.1, 0.25, Y0.astype(np.float64))
    out = gpu_matvec(op, X, 1.1, 0.25, Y0, dtype="f32")
    assert colmax_rel(out, ref) <= TOL32


def test_e2e_host_buffers_equal_device():
    h = random_case(1500, 32, lambda l: 16, 15)
    op = _op(h, nv_max=3)
    X = make_xy(h.perm, 3, 1, -1.0, 1.0)
    Y0 = make_xy(h.perm, 3, 2, -1.0, 1.0, stream=1)
    dev = gpu_matvec(op, X, 0.8, 0.2, Y0)
    Yh = Y0.copy()
    op.matvec_host(np.ascontiguousarray(X), Yh, 0.8, 0.2)
    assert np.array_equal(Yh, dev)


@pytest.mark.parametrize("dtype,nv,beta", [("f64", 16, 0.2), ("f64", 21, 0.0), ("f32", 16, 0.2)])
def test_e2e_pipelined_chunks(dtype, nv, beta, monkeypatch):
    """h2_matvec_host in two vector chunks (host-to-device of chunk 1 overlapping the matvec of
    chunk 0, device-to-host of chunk 0 overlapping chunk 1; forced on a small case): equal to the
    device-buffer matvec within rounding, and to the oracle."""
    monkeypatch.setenv("H2_E2E_MIN_MB", "0")
    h = random_case(3000, 32, lambda l: 16, 17)
    hh = h.astype(np.float32) if dtype == "f32" else h
    npdt = np.float32 if dtype == "f32" else np.float64
    op = _op(hh, nv_max=nv, dtype=dtype)
    X = make_xy(h.perm, nv, 3, -1.0, 1.0).astype(npdt)
    Y0 = make_xy(h.perm, nv, 4, -1.0, 1.0, stream=1).astype(npdt)
    dev = gpu_matvec(op, X, 0.7, beta, Y0, dtype)
    Yh = np.ascontiguousarray(Y0.copy())
    op.matvec_host(np.ascontiguousarray(X), Yh, 0.7, beta)
    tol = TOL32 if dtype == "f32" else 1e-13
    assert colmax_rel(Yh, dev) <= tol
    ref = oracle.matvec(hh.astype(np.float64), X.astype(np.float64), 0.7, beta, Y0.astype(np.float64))
    assert colmax_rel(Yh, ref) <= (TOL32 if dtype == "f32" else TOL64)


def test_single_leaf_and_all_dense():
    from h2gen import build_cluster_tree, dual_traversal, random_h2_data
    from h2gen.tree import uniform_points
    tr = build_cluster_tree(uniform_points(40, 2, 3), 64)   # q = 0: one dense block
    st = dual_traversal(tr, 0.9)
    h = random_h2_data(tr, st, [7], 3)
    X = make_xy(h.perm, 2, 1, -1.0, 1.0)
    assert colmax_rel(gpu_matvec(_op(h, nv_max=2), X, 1.0, 0.0, np.zeros_like(X)),
                      oracle.matvec(h, X)) <= TOL64
    tr = build_cluster_tree(uniform_points(800, 2, 4), 32)
    st = dual_traversal(tr, 0.9, all_dense=True)
    h = random_h2_data(tr, st, [9] * (tr.q + 1), 4)
    X = make_xy(h.perm, 2, 1, -1.0, 1.0)
    assert colmax_rel(gpu_matvec(_op(h, nv_max=2), X, 1.0, 0.0, np.zeros_like(X)),
                      oracle.matvec(h, X)) <= TOL64


def test_per_phase_trees_cfg1():
    """Y of a pure-low-rank operator (dense blocks zeroed) isolates upsweep + coupling + downsweep."""
    h = build_config("cfg1")
    h.D = np.zeros_like(h.D)
    X = make_xy(h.perm, 2, 5, -1.0, 1.0)
    ref = oracle.matvec(h, X)
    out = gpu_matvec(_op(h, nv_max=2), X, 1.0, 0.0, np.zeros_like(X))
    assert colmax_rel(out, ref) <= TOL64


@pytest.mark.slow
@pytest.mark.parametrize("nv", [1, 16])
def test_cfg2_full_size_sampled(nv):
    """The bench workload at its full size and launch configuration: sampled-row oracle on 2% of
    the leaves (exact arithmetic of those rows), alpha=1, beta=0."""
    h = build_config("cfg2")
    op = _op(h, nv_max=16)
    X = make_xy(h.perm, nv, 3, 0.0, 1.0)
    out = gpu_matvec(op, X, 1.0, 0.0, np.zeros_like(X))
    mask = np.zeros(1 << h.q, dtype=bool)
    mask[np.random.default_rng(0).choice(mask.size, mask.size // 50, replace=False)] = True
    mask[[0, -1]] = True
    ref = oracle.matvec(h, X, 1.0, 0.0, None, leaf_mask=mask)
    rows = np.concatenate([np.arange(h.leaf_ptr[i], h.leaf_ptr[i + 1]) for i in np.flatnonzero(mask)])
    assert colmax_rel(out[:, rows], ref[:, rows]) <= TOL64


def test_cfg3_structure_small():
    """cfg3's structure (3D Gaussian, k = 4^3 = 64, eta = 1.1; readings R5, R8, R9) at nv = 64 on
    a 16x16x32 grid (128 leaves): every element against the oracle, alpha and beta nonzero."""
    h = build_config("cfg3", points=("grid", (16, 16, 32)))
    assert h.ranks[-1] == 64 and h.dim == 3
    op = _op(h, nv_max=64)
    X = make_xy(h.perm, 64, 8, -1.0, 1.0)
    Y0 = make_xy(h.perm, 64, 8, -1.0, 1.0, stream=1)
    ref = oracle.matvec(h, X, 0.8, 1.5, Y0)
    out = gpu_matvec(op, X, 0.8, 1.5, Y0)
    assert colmax_rel(out, ref) <= TOL64


@pytest.mark.slow
def test_cfg3s_full_size_sampled():
    """bench.py --config cfg3s at its full size (64^3 points, nv = 64, nv_max = 64): sampled-row
    oracle on 2% of the leaves, alpha=1, beta=0."""
    h = build_config("cfg3", points=("grid", (64, 64, 64)))
    op = _op(h, nv_max=64)
    X = make_xy(h.perm, 64, 3, 0.0, 1.0)
    out = gpu_matvec(op, X, 1.0, 0.0, np.zeros_like(X))
    mask = np.zeros(1 << h.q, dtype=bool)
    mask[np.random.default_rng(1).choice(mask.size, mask.size // 50, replace=False)] = True
    mask[[0, -1]] = True
    ref = oracle.matvec(h, X, 1.0, 0.0, None, leaf_mask=mask)
    rows = np.concatenate([np.arange(h.leaf_ptr[i], h.leaf_ptr[i + 1]) for i in np.flatnonzero(mask)])
    assert colmax_rel(out[:, rows], ref[:, rows]) <= TOL64


@pytest.mark.parametrize("engine", ["warp", "cta"])
@pytest.mark.parametrize("N,m,k,nv,eta,seed", [
    (3000, 32, 16, 1, 0.9, 51), (3000, 32, 25, 3, 0.9, 52), (5000, 64, 25, 8, 0.9, 53),
    (5000, 64, 25, 16, 0.9, 54), (4000, 64, 36, 17, 0.9, 55), (4000, 64, 64, 33, 1.1, 56),
    (4000, 64, 64, 64, 1.1, 57), (2500, 48, 40, 20, 0.9, 58)])
def test_engines(engine, N, m, k, nv, eta, seed, monkeypatch):
    """Both FP64 engines on every shape class: the warp-task engine (H2_ENGINE=warp) and the
    CTA-tile engine (H2_ENGINE=cta: every block staged once in shared memory for all warps of
    the CTA), odd / even k, ragged leaves, nv inside and across the 16-vector chunks."""
    monkeypatch.setenv("H2_ENGINE", engine)
    h = random_case(N, m, lambda l: k, seed, eta=eta)
    X = make_xy(h.perm, nv, seed, -1.0, 1.0)
    Y0 = make_xy(h.perm, nv, seed + 1, -1.0, 1.0, stream=1)
    out = gpu_matvec(_op(h, nv_max=max(nv, 16)), X, -0.6, 1.3, Y0)
    ref = oracle.matvec(h, X, -0.6, 1.3, Y0)
    assert colmax_rel(out, ref) <= TOL64


def test_matvec_ld_larger_leading_dimensions():
    """h2_matvec_ld with ldx, ldy > n_local (include/h2.h): columns strided inside larger buffers;
    the padding between columns is neither read into the result nor written."""
    import torch
    h = random_case(3000, 32, lambda l: 12, 71)
    op = _op(h, nv_max=5)
    nv, N = 5, h.N
    ldx, ldy = N + 37, N + 64
    X = make_xy(h.perm, nv, 7, -1.0, 1.0)
    Y0 = make_xy(h.perm, nv, 8, -1.0, 1.0, stream=1)
    Xb = torch.full((nv * ldx,), float("nan"), dtype=torch.float64, device="cuda")
    Yb = torch.full((nv * ldy,), 123.0, dtype=torch.float64, device="cuda")
    for c in range(nv):
        Xb[c * ldx:c * ldx + N] = torch.from_numpy(X[c])
        Yb[c * ldy:c * ldy + N] = torch.from_numpy(Y0[c])
    op.matvec_ld(Xb, ldx, Yb, ldy, nv, -0.5, 0.25)
    torch.cuda.synchronize()
    Yh = Yb.cpu().numpy()
    out = np.stack([Yh[c * ldy:c * ldy + N] for c in range(nv)])
    assert colmax_rel(out, oracle.matvec(h, X, -0.5, 0.25, Y0)) <= TOL64
    pad = np.concatenate([Yh[c * ldy + N:(c + 1) * ldy] for c in range(nv)])
    assert np.all(pad == 123.0)


@pytest.mark.parametrize("engine", ["warp", "tcgen05"])
@pytest.mark.parametrize("N,m,k,nv,eta,seed", [
    (3000, 32, 16, 5, 0.9, 61), (5000, 64, 25, 8, 0.9, 62), (5000, 64, 25, 16, 0.9, 63),
    (4000, 64, 36, 17, 0.9, 64), (4000, 64, 64, 16, 1.1, 65), (2500, 48, 40, 33, 0.9, 66),
    (3000, 64, 64, 64, 1.1, 67), (3000, 64, 64, 41, 1.1, 68)])
def test_fp32_tensor_engine(engine, N, m, k, nv, eta, seed, monkeypatch):
    """FP32 at nv >= 5 runs 3xTF32 on the tensor cores -- the coupling rows on tcgen05.mma (TMEM
    accumulators, h2_umma.cuh) by default, everything on the mma.sync warp engine (Tf3) with
    H2_ENGINE=warp: within 1e-5 of the FP64 oracle on the FP32-rounded operator and vectors, ragged
    leaves, unaligned ranks (k = 25: 4-byte copies), nv inside and across the 8/16/32/64 chunks."""
    if engine == "warp":
        monkeypatch.setenv("H2_ENGINE", "warp")
    h = random_case(N, m, lambda l: k, seed, eta=eta).astype(np.float32)
    X = make_xy(h.perm, nv, seed, -1.0, 1.0).astype(np.float32).astype(np.float64)
    Y0 = make_xy(h.perm, nv, seed + 1, -1.0, 1.0, stream=1).astype(np.float32).astype(np.float64)
    out = gpu_matvec(_op(h, nv_max=max(nv, 16), dtype="f32"), X, -0.6, 1.3, Y0, "f32")
    ref = oracle.matvec(h.astype(np.float64), X, -0.6, 1.3, Y0)
    assert colmax_rel(out, ref) <= TOL32


def test_per_phase_xhat_yhat_trees():
    """the x^ and y^ trees the GPU leaves after a matvec, level by level, against
    brute force -- x^^l_s = V^{lT}_s x_s with the explicit level bases (upsweep: leaf projection +
    transfers), c^l_t = sum_s S_ts x^^l_s (coupling), y^^l = c^l + E y^^{l-1}_parent (downsweep, levels
    above the leaves; the FP64 leaf kernel applies the last transfer itself, so the leaf level holds
    c^q)."""
    from paper_2109_05451_b200._binding import H2_EXPORT_XHAT, H2_EXPORT_YHAT
    from tests.dense_assembly import explicit_bases
    h = random_case(1500, 32, lambda l: 8 + (l % 2), 21)
    nv = 2
    op = _op(h, nv_max=nv)
    X = make_xy(h.perm, nv, 7, -1.0, 1.0)
    gpu_matvec(op, X, 1.0, 0.0, np.zeros_like(X))
    VB = explicit_bases(h, "V")
    q = h.q
    xh_ref, c_ref = {}, {}
    for l in range(q + 1):
        k = h.ranks[l]
        sh = q - l
        xs = np.zeros((nv, 1 << l, k))
        for s in range(1 << l):
            r0, r1 = h.leaf_ptr[s << sh], h.leaf_ptr[(s + 1) << sh]
            xs[:, s, :] = (VB[(l, s)].T @ X[:, r0:r1].T).T
        xh_ref[l] = xs
        c = np.zeros((nv, 1 << l, k))
        rp, col = h.S_rowptr[l], h.S_col[l]
        for t in range(1 << l):
            for b in range(rp[t], rp[t + 1]):
                c[:, t, :] += (h.S[l][b].T @ xs[:, col[b], :].T).T
        c_ref[l] = c
    y_ref = {0: c_ref[0]}
    for l in range(1, q + 1):
        y_ref[l] = c_ref[l] + np.einsum("cij,nci->ncj", h.E[l], y_ref[l - 1][:, np.arange(1 << l) >> 1, :])
    for l in range(q + 1):
        k = h.ranks[l]
        got_x = op.export(H2_EXPORT_XHAT, l, nv * (1 << l) * k).reshape(nv, 1 << l, k)
        if np.abs(c_ref[l]).max() > 0 or l == q:      # levels whose x^ feeds a coupling or transfer
            assert np.abs(got_x - xh_ref[l]).max() <= 1e-12 * np.abs(xh_ref[l]).max(), ("x^", l)
        got_y = op.export(H2_EXPORT_YHAT, l, nv * (1 << l) * k).reshape(nv, 1 << l, k)
        want = c_ref[q] if l == q else y_ref[l]
        assert np.abs(got_y - want).max() <= 1e-12 * max(np.abs(want).max(), 1e-300), ("y^", l)
    op.close()
