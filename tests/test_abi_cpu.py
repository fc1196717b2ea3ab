"""C-ABI library checks that need no GPU: it loads, exports every symbol include/h2.h declares,
and h2_create's validation rejects bad descriptions before touching the device."""
import os
import re

import numpy as np
import pytest

import paper_2109_05451_b200 as pkg
from paper_2109_05451_b200._binding import H2Error
from paper_2109_05451_b200.operator import shard_arrays

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "h2.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(h2_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    lib = pkg.load_library()
    decl = declared_symbols()
    assert len(decl) >= 10
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(pkg.EXPORTS)
    assert b"sm_100a" in lib.h2_version()


def _small():
    from h2gen import build_cluster_tree, dual_traversal, random_h2_data
    from h2gen.tree import uniform_points
    tr = build_cluster_tree(uniform_points(300, 2, 1), 16)
    st = dual_traversal(tr, 0.9)
    return random_h2_data(tr, st, [8] * (tr.q + 1), 2)


def _create(kw, **over):
    kw = dict(kw)
    kw.update(over)
    return pkg.H2Operator(**kw)


def test_validation_errors_without_gpu():
    h = _small()
    kw, _ = shard_arrays(h, 0, 1)
    # leaf size above the supported 64
    with pytest.raises(H2Error) as e:
        _create(kw, leaf_size=65)
    assert e.value.code == pkg.H2_ERR_SHAPE
    # rank above 64
    with pytest.raises(H2Error) as e:
        _create(kw, level_rank=np.full(h.q + 1, 65, dtype=np.int32))
    assert e.value.code == pkg.H2_ERR_SHAPE
    # nv_max out of range
    with pytest.raises(H2Error) as e:
        _create(kw, nv_max=0)
    assert e.value.code == pkg.H2_ERR_SHAPE
    # non power-of-two ranks
    with pytest.raises(H2Error) as e:
        _create(kw, nranks=3, nccl_id=b"\0" * 128)
    assert e.value.code == pkg.H2_ERR_STRUCT
    # duplicate coupling block (t, s, l)
    l = max(range(h.q + 1), key=lambda l: h.S_col[l].size)
    bad_col = [c.copy() for c in kw["S_col"]]
    rp = kw["S_rowptr"][l]
    row = int(np.argmax(np.diff(rp)))
    bad_col[l][rp[row] + 1] = bad_col[l][rp[row]]
    with pytest.raises(H2Error) as e:
        _create(kw, S_col=bad_col)
    assert e.value.code == pkg.H2_ERR_STRUCT
    # leaf larger than m
    lp = kw["leaf_ptr"].copy()
    with pytest.raises(H2Error) as e:
        _create(kw, leaf_ptr=lp * 3, n_local=int(lp[-1] * 3))
    assert e.value.code == pkg.H2_ERR_STRUCT
    # column out of range
    bad_col = [c.copy() for c in kw["S_col"]]
    bad_col[l][-1] = 1 << l
    with pytest.raises(H2Error) as e:
        _create(kw, S_col=bad_col)
    assert e.value.code == pkg.H2_ERR_STRUCT


def test_shard_arrays_partition():
    """Rank shards partition the rows, dense blocks and branch-level coupling blocks exactly."""
    h = _small()
    for P in (1, 2, 4):
        rows, nd, ns = [], 0, 0
        for p in range(P):
            kw, (r0, r1) = shard_arrays(h, p, P)
            rows.append((r0, r1))
            nd += kw["D_col"].size
            ns += sum(c.size for l, c in enumerate(kw["S_col"]) if (1 << l) >= P)
        assert rows[0][0] == 0 and rows[-1][1] == h.N
        assert all(rows[i][1] == rows[i + 1][0] for i in range(P - 1))
        assert nd == h.n_D
        assert ns == sum(c.size for l, c in enumerate(h.S_col) if (1 << l) >= P)
