"""Full-size parity of the BASELINE.json workloads in the launch configuration bench.py times
(nv_max = the workload's largest nv, alpha = 1, beta = 0, X ~ U[0,1) from the counter RNG): the
sampled-row oracle (SURVEY.md §8(c) "full-size parity beyond host RAM" — exact arithmetic of the
sampled leaves' rows, full upsweep) on >= 2 % of the leaves, plus the first and last leaf.

Tolerances: north_star's relative 2-norm per column, 1e-12 in FP64; FP32 against the FP64 oracle
on the FP32-rounded operator and X, 1e-5."""
import numpy as np
import pytest

import oracle
from h2gen import make_xy
from h2gen.configs import build_config, CONFIGS
from tests.gpu_util import colmax_rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2109_05451_b200 import load_library
    load_library()
    oracle.set_threads(0)


def sampled_parity(name, dtype, nv, frac=0.02, seed=5):
    import torch
    from paper_2109_05451_b200 import operator_from_h2data
    h = build_config(name)
    nvmax = max(CONFIGS[name]["nvs"])
    hx = h if dtype == "f64" else h.astype(np.float32).astype(np.float64)
    X = make_xy(h.perm, nv, seed, 0.0, 1.0)
    if dtype == "f32":
        X = X.astype(np.float32).astype(np.float64)
    op = operator_from_h2data(h, dtype=dtype, nv_max=nvmax)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    Xd = torch.from_numpy(X).to("cuda", tdt)
    Yd = torch.zeros_like(Xd)
    op.matvec(Xd, Yd, 1.0, 0.0)
    torch.cuda.synchronize()
    out = Yd.double().cpu().numpy()
    op.close()
    del op, Xd, Yd
    nleaf = 1 << h.q
    mask = np.zeros(nleaf, dtype=bool)
    mask[np.random.default_rng(seed).choice(nleaf, max(2, int(nleaf * frac)), replace=False)] = True
    mask[[0, -1]] = True
    ref = oracle.matvec(hx, X, 1.0, 0.0, None, leaf_mask=mask)
    rows = np.concatenate([np.arange(h.leaf_ptr[i], h.leaf_ptr[i + 1]) for i in np.flatnonzero(mask)])
    assert np.all(np.isfinite(out))
    return colmax_rel(out[:, rows], ref[:, rows])


@pytest.mark.slow
def test_cfg3_full_size_sampled():
    """cfg3 at its real size: 128^3 = 2^21 points, 3D Gaussian, k = 64, eta = 1.1, nv = 64, FP64
    (BASELINE configs[2]; 742,490 coupling + 195,872 dense blocks, 37 GB)."""
    assert sampled_parity("cfg3", "f64", 64) <= 1e-12


@pytest.mark.slow
def test_cfg4_full_size_sampled():
    """cfg4 at its P = 1 size: the FD operator on the 1448^2 interior grid (ragged leaves), k = 36,
    nv = 1, FP64 (BASELINE configs[3])."""
    assert sampled_parity("cfg4", "f64", 1) <= 1e-12


@pytest.mark.slow
@pytest.mark.parametrize("dtype,tol", [("f64", 1e-12), ("f32", 1e-5)])
def test_cfg5_full_size_sampled(dtype, tol):
    """cfg5 at its P = 1 size: 3D exp kernel on 128^3 points, k = 64, nv = 16, FP64 and FP32
    (BASELINE configs[4])."""
    assert sampled_parity("cfg5", dtype, 16) <= tol
