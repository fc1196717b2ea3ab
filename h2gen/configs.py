"""The BASELINE.json workloads (SURVEY.md §8(d) "Concrete synthetic inputs"); seed 210905451."""
from .tree import build_cluster_tree, grid_points, uniform_points
from .structure import dual_traversal
from .kernels import Kernel
from .h2data import build_h2

SEED = 210905451

CONFIGS = {
    # name: points, dim, m, p (k = p^dim), eta, kernel, nvs, dtype
    "cfg1": dict(points=("uniform", 4096, 2), m=32, p=4, eta=0.9, kernel=("exp", 0.1), nvs=(1,),
                 desc="2D exp-covariance kernel, N=4096 uniform points, leaf 32, Chebyshev rank 16, nv=1, FP64, 1 GPU"),
    "cfg1grid": dict(points=("grid", (64, 64)), m=32, p=4, eta=0.9, kernel=("exp", 0.1), nvs=(1,),
                     desc="cfg1 grid variant (64x64)"),
    "cfg2": dict(points=("grid", (1024, 1024)), m=64, p=5, eta=0.9, kernel=("exp", 0.1), nvs=(1, 16),
                 desc="2D exp-covariance kernel, N=1M points, leaf 64, rank 25, nv=1 and nv=16, FP64, 1 GPU"),
    "cfg3": dict(points=("grid", (128, 128, 128)), m=64, p=4, eta=1.1, kernel=("gaussian", 0.2), nvs=(64,),
                 desc="3D Gaussian kernel, N=2M points, leaf 64, rank 64, nv=64, FP64"),
    "cfg5": dict(points=("grid", (128, 128, 128)), m=64, p=4, eta=1.1, kernel=("exp", 0.2), nvs=(16,),
                 desc="3D exp-covariance kernel, 2M points per GPU, leaf 64, rank 64, nv=16"),
    # the paper's own 2D set at 2^19 points: structure pin C_sp = 17
    "paper2d": dict(points=("grid", (1024, 512)), m=64, p=8, eta=0.9, kernel=("exp", 0.1), nvs=(1,),
                    desc="paper 2D set, N=2^19, m=64, k=64, eta=0.9"),
}


def config_params(name):
    return CONFIGS[name]


def make_points(spec, seed=SEED):
    if spec[0] == "uniform":
        return uniform_points(spec[1], spec[2], seed)
    return grid_points(spec[1])


def build_config(name, seed=SEED, **override):
    c = dict(CONFIGS[name])
    c.update(override)
    pts = make_points(c["points"], seed)
    tree = build_cluster_tree(pts, c["m"])
    st = dual_traversal(tree, c["eta"])
    kname, ell = c["kernel"]
    return build_h2(tree, st, Kernel(kname, ell=ell, p=c["p"]), c["p"])
