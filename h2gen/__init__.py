"""h2gen — seeded synthetic INPUT generator for the H² matvec (test/bench infrastructure).

This package builds the operator data the method runs on (cluster tree, block
structure, Chebyshev-interpolation bases/transfers/couplings, dense near-field
blocks) and the seeded X/Y multivectors. It holds none of the matvec's
arithmetic (no upsweep / coupling multiply / downsweep / dense product): both
the CPU oracle (`oracle/`) and the CUDA path (`paper_2109_05451_b200`) consume
what it produces, and neither is imported here.

Storage convention for every small matrix A (r x c): column-major, i.e. a batch
of them is a C-contiguous numpy array of shape (batch, c, r) with
arr[b, j, i] = A_b[i, j].  See DESIGN.md "Data layout".
"""
from .tree import ClusterTree, build_cluster_tree
from .structure import BlockStructure, dual_traversal
from .h2data import H2Data, build_h2, random_h2_data, poly_kernel_apply
from .rng import counter_uniform, make_xy
from .configs import CONFIGS, SEED, config_params, build_config

__all__ = [
    "ClusterTree", "build_cluster_tree", "BlockStructure", "dual_traversal",
    "H2Data", "build_h2", "random_h2_data", "poly_kernel_apply",
    "counter_uniform", "make_xy", "CONFIGS", "SEED", "config_params", "build_config",
]
