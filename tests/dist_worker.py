"""Multi-GPU parity worker (launched by torchrun, one rank per GPU, NCCL):
every rank builds the same global problem, creates its block-row shard through the C ABI, runs
the distributed matvec, and rank 0 compares the concatenated Y with the CPU oracle and with the
single-GPU result.  Exit code 0 = pass.  Cases include a structure with top-tree (root branch)
couplings (eta = 3) so the replicated top-tree path runs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch
import torch.distributed as dist


def main():
    import oracle
    import paper_2109_05451_b200 as pkg
    from h2gen import build_config, make_xy, build_cluster_tree, dual_traversal, random_h2_data
    from h2gen.tree import uniform_points
    from paper_2109_05451_b200.operator import operator_from_h2data
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from tests.gpu_util import with_root_coupling
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lr)
    dev = torch.device("cuda", lr)
    dist.init_process_group("nccl", device_id=dev)
    pkg.load_library()
    from paper_2109_05451_b200.operator import broadcast_nccl_id

    def rand(N, m, k, eta, seed):
        tr = build_cluster_tree(uniform_points(N, 2, seed), m)
        st = dual_traversal(tr, eta)
        return random_h2_data(tr, st, [k] * (tr.q + 1), seed)

    cases = [("cfg1", build_config("cfg1"), 1, "f64"),
             ("rand-k25-nv16", rand(6000, 64, 25, 0.9, 5), 16, "f64"),
             ("rand-k36-nv3", rand(4000, 32, 36, 0.9, 6), 3, "f64"),
             ("rand-k25-nv20-chunks", rand(5000, 64, 25, 0.9, 8), 20, "f64"),
             ("rand-k16-fp32-nv5", rand(4000, 32, 16, 0.9, 9), 5, "f32"),
             ("top-tree-eta3", rand(5000, 32, 16, 3.0, 7), 2, "f64"),
             ("top-tree-root-block", with_root_coupling(rand(3000, 32, 12, 0.9, 12)), 4, "f64")]
    fails = 0
    for name, h, nv, dt in cases:
        if dt == "f32":
            h = h.astype(np.float32)
        print(f"[rank {rank}] case {name}: create", flush=True)
        op = operator_from_h2data(h, rank=rank, nranks=world, nccl_id=broadcast_nccl_id(dev), nv_max=nv, dtype=dt)
        print(f"[rank {rank}] case {name}: created", flush=True)
        r0, r1 = op.row_range
        npdt = np.float64 if dt == "f64" else np.float32
        X = make_xy(h.perm, nv, 11, -1.0, 1.0).astype(npdt)
        Y0 = make_xy(h.perm, nv, 12, -1.0, 1.0, stream=1).astype(npdt)
        Xd = torch.from_numpy(np.ascontiguousarray(X[:, r0:r1])).to(dev)
        Yd = torch.from_numpy(np.ascontiguousarray(Y0[:, r0:r1])).to(dev)
        for rep in range(3):                          # eager, then captured-graph calls
            Yd.copy_(torch.from_numpy(np.ascontiguousarray(Y0[:, r0:r1])))
            op.matvec(Xd, Yd, 0.75, -0.5)
            torch.cuda.synchronize()
            print(f"[rank {rank}] case {name}: call {rep} done", flush=True)
        pc = op.plan_counts()
        parts = [None] * world
        dist.all_gather_object(parts, (r0, r1, Yd.cpu().numpy(), pc))
        if rank == 0:
            Y = np.concatenate([p[2] for p in sorted(parts, key=lambda p: p[0])], axis=1)
            ref = oracle.matvec(h.astype(np.float64) if dt == "f32" else h, X.astype(np.float64), 0.75, -0.5,
                                Y0.astype(np.float64))
            Y = Y.astype(np.float64)
            err = max(np.linalg.norm(Y[i] - ref[i]) / np.linalg.norm(ref[i]) for i in range(nv))
            root = sum(p[3]["root_S"] for p in parts)
            off = sum(p[3]["offdiag_S"] for p in parts)
            ok = err <= (1e-12 if dt == "f64" else 1e-5)
            fails += 0 if ok else 1
            print(f"[dist P={world}] {name}: rel err {err:.2e} offdiag_S={off} root_S(all ranks)={root} "
                  f"{'OK' if ok else 'FAIL'}", flush=True)
            # eta = 3 has root-branch couplings only at P >= 4 (at P = 2 the top tree is the root
            # alone); the root-block case has them at every P >= 2
            if ((name == "top-tree-root-block" and world > 1) or (name == "top-tree-eta3" and world >= 4)) \
                    and root == 0:
                print(f"[dist] FAIL: {name} has no root-branch couplings at P={world}", flush=True)
                fails += 1
        op.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
