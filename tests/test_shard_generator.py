"""The shard-aware generator (h2gen/shard.py, used by bench.py for P > 1 without a global
operator) must produce exactly the per-rank view that slicing the global operator gives
(paper_2109_05451_b200.operator.shard_arrays(build_h2(...))), so the multi-GPU bench inputs are
the same problem the oracle checks.  Host-only."""
import numpy as np
import pytest

from h2gen.configs import build_structure
from h2gen.h2data import build_h2
from h2gen.shard import build_h2_shard
from paper_2109_05451_b200.operator import shard_arrays


def _same(a, b, key):
    if isinstance(a, list):
        assert len(a) == len(b), key
        for i, (x, y) in enumerate(zip(a, b)):
            _same(x, y, f"{key}[{i}]")
    elif a is None or b is None:
        assert a is None and b is None, key
    elif isinstance(a, np.ndarray) or isinstance(b, np.ndarray):
        assert np.array_equal(np.asarray(a), np.asarray(b)), key
    else:
        assert a == b, key


@pytest.mark.parametrize("name,override", [
    ("cfg1", {}),
    ("cfg3", {"points": ("grid", (8, 16, 16))}),
    ("cfg4", {"points": ("fdgrid", 64)}),
])
@pytest.mark.parametrize("P", [2, 4])
def test_shard_generator_equals_sliced_global(name, override, P):
    tree, st, kern, c = build_structure(name, 1, **override)
    h = build_h2(tree, st, kern, c["p"])
    for rank in range(P):
        want, rows_w = shard_arrays(h, rank, P)
        got, rows_g = build_h2_shard(tree, st, kern, c["p"], rank, P)
        assert rows_w == rows_g
        assert set(want) == set(got)
        for key in want:
            _same(want[key], got[key], key)
