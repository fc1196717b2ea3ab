"""Multi-rank host logic without a GPU: the compressed off-diagonal node lists of the C-ABI plan
census on the paper's worked example, and a world_size-2 gloo run in which
two processes exchange their request lists and check them against each other and against an
independent computation from the global structure."""
import os
import socket

import numpy as np
import pytest

import paper_2109_05451_b200 as pkg
from paper_2109_05451_b200.operator import shard_arrays, held_range


def _paper_example_view():
    """A hand-built 4-rank structure whose level-4 off-diagonal columns for rank 0 are the
    paper's Fig. compressed_vnodes example (the figure itself is lost: format only)."""
    from h2gen import build_cluster_tree, dual_traversal, random_h2_data
    from h2gen.tree import uniform_points
    tr = build_cluster_tree(uniform_points(16 * 8, 2, 1), 8)        # q = 4, 16 leaves
    st = dual_traversal(tr, 0.9)
    h = random_h2_data(tr, st, [4] * (tr.q + 1), 1)
    q = tr.q
    assert q == 4
    # replace the coupling structure of level 4: rows 0..3 (rank 0) -> columns {5, 6} (rank 1)
    # and {12, 13, 14} (rank 3); rank 2 is never referenced
    rows = {0: [5, 12], 1: [6, 13, 14], 2: [], 3: [5]}
    rp, col = [0], []
    for t in range(16):
        c = sorted(rows.get(t, []))
        col += c
        rp.append(len(col))
    h.S_rowptr[q] = np.array(rp, dtype=np.int64)
    h.S_col[q] = np.array(col, dtype=np.int32)
    h.S[q] = np.zeros((len(col), 4, 4))
    return h


def test_compressed_node_format_paper_example(golden):
    ex = golden["compressed_nodes_example"]
    h = _paper_example_view()
    kw, _ = shard_arrays(h, ex["rank"], ex["P"])
    pid, ptr, nodes = pkg.plan_census(4, **kw)
    assert list(pid) == ex["pid"]
    assert list(ptr) == ex["nodes_ptr"]
    assert list(nodes) == ex["nodes"]


def _needed_from_global(h, rank, P, level):
    """Independent reference: unique remote columns of rank's rows at `level` per owner."""
    a, b = held_range(level, rank, P)
    rp, col = h.S_rowptr[level], h.S_col[level]
    cols = set(int(c) for c in col[rp[a]:rp[b]])
    C = P.bit_length() - 1
    if level < C:
        return {}
    w = 1 << (level - C)
    out = {}
    for c in sorted(cols):
        o = c // w
        if o != rank:
            out.setdefault(o, []).append(c)
    return out


def test_census_matches_independent_computation():
    from h2gen import build_config
    h = build_config("cfg1")
    for P in (2, 4):
        for rank in range(P):
            kw, _ = shard_arrays(h, rank, P)
            for l in range(h.q + 1):
                pid, ptr, nodes = pkg.plan_census(l, **kw)
                ref = _needed_from_global(h, rank, P, l)
                got = {int(p): list(nodes[ptr[i]:ptr[i + 1]]) for i, p in enumerate(pid)}
                assert got == ref, (P, rank, l)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q_out):
    import torch.distributed as dist
    from h2gen import build_config
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h = build_config("cfg1")
        kw, (r0, r1) = shard_arrays(h, rank, world)
        # every rank's request lists (all levels + halo), exchanged like h2_create does at setup
        reqs = {}
        for l in list(range(h.q + 1)) + [-1]:
            pid, ptr, nodes = pkg.plan_census(l, **kw)
            for i, p in enumerate(pid):
                reqs.setdefault(int(p), []).append((l, [int(x) for x in nodes[ptr[i]:ptr[i + 1]]]))
        gathered = [None] * world
        dist.all_gather_object(gathered, reqs)
        # what peers ask from me must be mine
        C = world.bit_length() - 1
        ok = True
        for peer, r in enumerate(gathered):
            for l, nodes in r.get(rank, []):
                lev = h.q if l < 0 else l
                a, b = held_range(lev, rank, world)
                ok &= all(a <= n < b for n in nodes)
        # row ranges partition [0, N)
        rows = [None] * world
        dist.all_gather_object(rows, (r0, r1))
        ok &= rows[0][0] == 0 and rows[-1][1] == h.N and all(rows[i][1] == rows[i + 1][0] for i in range(world - 1))
        q_out.put((rank, bool(ok), sum(len(n) for rr in gathered for lst in rr.values() for _, n in lst)))
    finally:
        dist.destroy_process_group()


def test_gloo_world_size_2_request_exchange():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res)
    assert res[0][2] == res[1][2] > 0
