"""Counter-based RNG for X / Y (values indexed by (original point id, column)
so that any rank split of the tree-ordered rows sees identical data)."""
import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(z):
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z += np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def counter_uniform(seed, ids, col, lo=0.0, hi=1.0):
    """U[lo,hi) doubles, one per entry of `ids` (original point ids), for column `col`."""
    ids = np.asarray(ids, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = _splitmix64(np.uint64(seed) ^ _splitmix64(np.asarray([col], dtype=np.uint64)))
        u = _splitmix64(ids * np.uint64(0xD1B54A32D192ED03) ^ key)
    return lo + (hi - lo) * ((u >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0))


def make_xy(perm, nv, seed, lo=0.0, hi=1.0, stream=0):
    """N x nv column-major multivector in TREE order (row r = original point perm[r]).

    Returned as a numpy array of shape (nv, N) (C-contiguous == N x nv column-major).
    `stream` separates independent draws (e.g. X uses 0, Y uses 1)."""
    perm = np.asarray(perm, dtype=np.uint64)
    out = np.empty((nv, perm.size), dtype=np.float64)
    for c in range(nv):
        out[c] = counter_uniform(seed + 7919 * stream, perm, c, lo, hi)
    return out
