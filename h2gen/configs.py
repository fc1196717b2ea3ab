"""The BASELINE.json workloads (SURVEY.md §8(d) "Concrete synthetic inputs"); seed 210905451.

A workload names a point set, a kernel, the leaf size m, the Chebyshev order p (k = p^dim), the
admissibility eta, the vector counts and the precisions.  Multi-GPU scaling follows SURVEY.md
§8(d)/(e):
  weak    P x the base point count (the shorter grid side doubled per factor 2; cfg4 uses its own
          n x n FD grids with n = 1448 / 2048 / 2896 / 4096 for P = 1 / 2 / 4 / 8),
  strong  the base problem split over P ranks.
"""
import numpy as np

from .tree import build_cluster_tree, grid_points, uniform_points, fd_grid_points
from .structure import dual_traversal
from .kernels import Kernel
from .h2data import build_h2

SEED = 210905451

CONFIGS = {
    # name: points, m, p (k = p^dim), eta, kernel, nvs, dtypes, scaling
    "cfg1": dict(points=("uniform", 4096, 2), m=32, p=4, eta=0.9, kernel=("exp", 0.1), nvs=(1,),
                 dtypes=("f64",), scaling="weak",
                 desc="2D exp-covariance kernel, N=4096 uniform points, leaf 32, Chebyshev rank 16, nv=1, FP64, 1 GPU"),
    "cfg1grid": dict(points=("grid", (64, 64)), m=32, p=4, eta=0.9, kernel=("exp", 0.1), nvs=(1,),
                     dtypes=("f64",), scaling="weak", desc="cfg1 grid variant (64x64)"),
    "cfg2": dict(points=("grid", (1024, 1024)), m=64, p=5, eta=0.9, kernel=("exp", 0.1), nvs=(1, 16),
                 dtypes=("f64",), scaling="weak",
                 desc="2D exp-covariance kernel, N=1M points, leaf 64, rank 25, nv=1 and nv=16, FP64"),
    # 3D Gaussian exp(-(r/0.2)^2) (reading R9), eta = 1.1 (reading R5)
    "cfg3": dict(points=("grid", (128, 128, 128)), m=64, p=4, eta=1.1, kernel=("gaussian", 0.2), nvs=(64,),
                 dtypes=("f64",), scaling="strong",
                 desc="3D Gaussian kernel, N=2M points (128^3 grid), leaf 64, rank 64, eta 1.1, nv=64, FP64"),
    # cfg3's structure at 1/8 the size (round-1 proxy, kept for quick parity / profiling runs)
    "cfg3s": dict(points=("grid", (64, 64, 64)), m=64, p=4, eta=1.1, kernel=("gaussian", 0.2), nvs=(64,),
                  dtypes=("f64",), scaling="strong",
                  desc="3D Gaussian kernel (cfg3 structure), N=64^3 points, leaf 64, rank 64, eta 1.1, nv=64, FP64"),
    # integral fractional diffusion operator K_ij = -2 sqrt(k_i k_j) / r^(2+2beta) (reading R10) on
    # the interior vertex grid of [-1,1]^2; k = 6^2 = 36 ("6x6")
    "cfg4": dict(points=("fdgrid", 1448), m=64, p=6, eta=0.9, kernel=("fd", 0.75), nvs=(1,),
                 dtypes=("f64",), scaling="weak",
                 desc="2D variable-diffusivity fractional diffusion operator (beta 0.75), 1448^2 ~ 2M DOF per GPU, "
                      "leaf 64, rank 36, nv=1, FP64"),
    "cfg5": dict(points=("grid", (128, 128, 128)), m=64, p=4, eta=1.1, kernel=("exp", 0.2), nvs=(16,),
                 dtypes=("f64", "f32"), scaling="weak",
                 desc="3D exp-covariance kernel, 2M points per GPU, leaf 64, rank 64, eta 1.1, nv=16, FP64 and FP32"),
    # the paper's own 2D set at 2^19 points: structure pin C_sp = 17
    "paper2d": dict(points=("grid", (1024, 512)), m=64, p=8, eta=0.9, kernel=("exp", 0.1), nvs=(1,),
                    dtypes=("f64",), scaling="weak", desc="paper 2D set, N=2^19, m=64, k=64, eta=0.9"),
}

FD_WEAK_N = {1: 1448, 2: 2048, 4: 2896, 8: 4096}   # SURVEY.md §8(d) cfg4 grids


def config_params(name):
    return CONFIGS[name]


def grid_for(base, P):
    """Weak-scaling grid: P x base points, doubling the shortest side per factor 2."""
    dims = list(base)
    n = P
    while n > 1:
        i = int(np.argmin(dims))
        dims[i] *= 2
        n //= 2
    return tuple(dims)


def make_points(spec, seed=SEED, P=1, weak=False):
    """Point set of a workload; weak=True scales it to P GPUs (module docstring)."""
    if spec[0] == "uniform":
        return uniform_points(spec[1] * (P if weak else 1), spec[2], seed)
    if spec[0] == "fdgrid":
        n = spec[1]
        if weak and P > 1:
            n = FD_WEAK_N[P] if n == FD_WEAK_N[1] and P in FD_WEAK_N else int(round(n * np.sqrt(P)))
        return fd_grid_points(n)
    return grid_points(grid_for(spec[1], P) if weak else spec[1])


def make_kernel(c):
    kname, par = c["kernel"]
    if kname == "fd":
        return Kernel("fd", beta=par)
    return Kernel(kname, ell=par, p=c["p"])


def build_structure(name, P=1, seed=SEED, **override):
    """(tree, block structure, kernel, config) of workload `name` at P GPUs (its own scaling)."""
    c = dict(CONFIGS[name])
    c.update(override)
    pts = make_points(c["points"], seed, P, weak=(c["scaling"] == "weak"))
    tree = build_cluster_tree(pts, c["m"])
    st = dual_traversal(tree, c["eta"])
    return tree, st, make_kernel(c), c


def build_config(name, seed=SEED, **override):
    tree, st, kern, c = build_structure(name, 1, seed, **override)
    return build_h2(tree, st, kern, c["p"])
