"""The .h2m flat file (layout in include/h2.h and h2gen/h2m.py): the generator
writes it, the oracle reads it back with its own reader (oracle/h2m.py), the library parses its
header without a GPU (h2_file_info), and -- on a GPU -- h2_create_from_file builds the same
operator (every rank reading only its own view)."""
import os

import numpy as np
import pytest

import oracle
from oracle.h2m import read_h2m
from h2gen import build_config, make_xy
from h2gen.h2m import write_h2m
from tests.gpu_util import colmax_rel, random_case


def _eq(a, b):
    if isinstance(a, list):
        return len(a) == len(b) and all(_eq(x, y) for x, y in zip(a, b))
    if a is None or b is None:
        return a is None and b is None
    return np.array_equal(np.asarray(a), np.asarray(b))


FIELDS = ["leaf_ptr", "U_leaf", "V_leaf", "E", "F", "S_rowptr", "S_col", "S", "D_rowptr", "D_col", "D", "perm", "points"]


@pytest.mark.parametrize("which", ["cfg1", "random-unsym"])
def test_roundtrip_oracle_reader(tmp_path, which):
    h = build_config("cfg1") if which == "cfg1" else random_case(700, 16, lambda l: 4 + l % 5, 31)
    path = str(tmp_path / "op.h2m")
    write_h2m(path, h, seed=210905451)
    r = read_h2m(path)
    assert (r.N, r.m, r.q, r.dim, list(r.ranks)) == (h.N, h.m, h.q, h.dim, list(h.ranks))
    for f in FIELDS:
        assert _eq(getattr(r, f), getattr(h, f)), f
    assert (r.V_leaf is r.U_leaf) == (h.V_leaf is h.U_leaf)
    X = make_xy(h.perm, 2, 3, -1.0, 1.0)
    assert np.array_equal(oracle.matvec(r, X, 1.0, 0.0), oracle.matvec(h, X, 1.0, 0.0))


def test_library_reads_header_without_gpu(tmp_path):
    from paper_2109_05451_b200 import H2Error
    from paper_2109_05451_b200._binding import file_info
    h = build_config("cfg1")
    path = str(tmp_path / "cfg1.h2m")
    write_h2m(path, h)
    info = file_info(path)
    assert info == {"N": h.N, "dim": 2, "m": h.m, "q": h.q, "dtype": 0, "n_S": h.n_S, "n_D": h.n_D, "k": h.ranks[-1]}
    with open(path, "r+b") as f:                 # truncated file -> structural error
        f.truncate(os.path.getsize(path) - 4096)
    with pytest.raises(H2Error):
        file_info(path)
    with pytest.raises(H2Error):
        file_info(str(tmp_path / "missing.h2m"))


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 2, 4])
def test_create_from_file_matches_oracle(tmp_path, P):
    import torch
    from paper_2109_05451_b200 import H2Operator, load_library
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    load_library()
    h = random_case(3000, 32, lambda l: 9 + l % 4, 41)
    path = str(tmp_path / "rand.h2m")
    write_h2m(path, h)
    X = make_xy(h.perm, 3, 5, -1.0, 1.0)
    Y0 = make_xy(h.perm, 3, 6, -1.0, 1.0, stream=1)
    ref = oracle.matvec(read_h2m(path), X, 0.5, 2.0, Y0)
    if P == 1:
        op = H2Operator.from_file(path, nv_max=4)
        Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y0.copy()).cuda()
        op.matvec(Xd, Yd, 0.5, 2.0)
        torch.cuda.synchronize()
        out = Yd.cpu().numpy()
        op.close()
    else:
        # every rank reads its own view from the file (h2_group_create_from_file)
        from paper_2109_05451_b200 import H2Group
        grp = H2Group(None, path=path, P=P, nv_max=4)
        lp = np.asarray(h.leaf_ptr)
        w = (1 << h.q) // P
        rows = [(int(lp[o * w]), int(lp[(o + 1) * w])) for o in range(P)]
        assert [b - a for a, b in rows] == grp.n_local
        Xs = [torch.from_numpy(np.ascontiguousarray(X[:, a:b])).cuda() for a, b in rows]
        Ys = [torch.from_numpy(np.ascontiguousarray(Y0[:, a:b])).cuda() for a, b in rows]
        grp.matvec(Xs, Ys, 0.5, 2.0)
        torch.cuda.synchronize()
        out = np.concatenate([y.cpu().numpy() for y in Ys], axis=1)
        grp.close()
    assert colmax_rel(out, ref) <= 1e-12
