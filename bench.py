#!/usr/bin/env python
"""bench.py — H² matvec throughput on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]

One STEP = one pass of the whole hot path (upsweep, coupling, downsweep, dense, epilogue) for
every nv the workload names (cfg2: nv=1 and nv=16), on inputs already resident in HBM.
N=1: BASELINE.json configs[1] (cfg2, 1M points, FP64).  N>1 (torchrun): weak scaling, each rank
holds a 1M-point branch of an N x 1M-point grid; the off-diagonal x^ / x halo exchange runs
over NCCL inside every matvec.  Timing: CUDA events on the launching stream, barrier + device
sync on both sides, max over ranks.  Rank 0 prints one JSON line.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "H2 matvec GFLOP/s per GPU and ms/matvec (nv=1,16,64) at 1/2/4/8 B200"
WORKLOADS = {
    "cfg2": dict(desc="2D exp-covariance kernel, N=1M points, leaf 64, rank 25, nv=1 and nv=16, FP64",
                 base=(1024, 1024), m=64, p=5, eta=0.9, kernel=("exp", 0.1), nvs=(1, 16), dtype="f64"),
    "cfg1": dict(desc="2D exp-covariance kernel, N=4096 uniform points, leaf 32, Chebyshev rank 16, nv=1, FP64",
                 base=None, m=32, p=4, eta=0.9, kernel=("exp", 0.1), nvs=(1,), dtype="f64"),
    # cfg3's structure (3D Gaussian, leaf 64, k = 4^3 = 64, eta = 1.1, nv = 64; reading R5/R9) on a
    # 64^3 grid: the compute-bound regime on one GPU without the 37 GB operator of the 128^3 case
    "cfg3s": dict(desc="3D Gaussian kernel (cfg3 structure), N=64^3=262144 grid points, leaf 64, rank 64, "
                       "eta 1.1, nv=64, FP64",
                  base=(64, 64, 64), m=64, p=4, eta=1.1, kernel=("gaussian", 0.2), nvs=(64,), dtype="f64"),
}


def grid_for(base, P):
    """Weak-scaling grid: P x base points, doubling the shorter side (longest side = 1)."""
    dims = list(base)
    n = P
    while n > 1:
        i = int(np.argmin(dims))
        dims[i] *= 2
        n //= 2
    return tuple(dims)


def fp64_peak():
    """Measured FP64 DMMA ceiling: cuBLAS DGEMM 8192^3 on this pool's B200 (profiles/peaks_b200_r01.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "peaks_b200_r01.json")) as f:
            return float(json.load(f)["gemm_float64_tflops"]), "measured cuBLAS DGEMM (profiles/peaks_b200_r01.json)"
    except Exception:
        return 40.0, "nominal B200 FP64 tensor 40 TFLOP/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None

    def __enter__(self):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.f.seek(0)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        busy = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rk = int(os.environ.get("RANK", "0"))
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rk, lr


def build_problem(wl, P, rank, with_global):
    from h2gen import build_cluster_tree, dual_traversal, SEED
    from h2gen.kernels import Kernel
    from h2gen.tree import grid_points, uniform_points
    from h2gen.shard import build_h2_shard
    from h2gen.h2data import build_h2
    if wl["base"] is None:
        pts = uniform_points(4096, 2, SEED)
    else:
        pts = grid_points(grid_for(wl["base"], P))
    tree = build_cluster_tree(pts, wl["m"])
    st = dual_traversal(tree, wl["eta"])
    kern = Kernel(wl["kernel"][0], ell=wl["kernel"][1])
    if with_global:
        h = build_h2(tree, st, kern, wl["p"])
        from paper_2109_05451_b200.operator import shard_arrays
        kw, rows = shard_arrays(h, rank, P)
        return tree, st, h, kw, rows
    kw, rows = build_h2_shard(tree, st, kern, wl["p"], rank, P)
    return tree, st, None, kw, rows


def run_reference(args, wl, emit):
    """--impl reference: the CPU oracle (oracle/, plain C FP64, single thread) on the same
    workload, one full step (every nv) per timed step; rank 0 only."""
    ws, rk, _ = dist_env()
    if rk != 0:
        return
    import oracle
    from h2gen import make_xy, SEED
    _, _, h, _, _ = build_problem(wl, 1, 0, True)
    prep = oracle.prepare(h)
    Xs = {nv: make_xy(h.perm, nv, SEED) for nv in wl["nvs"]}
    flops = sum(h.flops(nv) for nv in wl["nvs"])

    def step():
        for nv in wl["nvs"]:
            oracle.matvec(h, Xs[nv], 1.0, 0.0, None, prepared=prep)
    for _ in range(args.warmup):
        step()
    t = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        t.append(time.perf_counter() - t0)
    sec = sum(t) / len(t)
    val = flops / sec / 1e9
    out = {"metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": wl["dtype"], "data": "synthetic",
           "config": {"workload": f"{args.config}: {wl['desc']}", "N": int(h.N), "nvs": list(wl["nvs"])},
           "impl": "reference",
           "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
                            "sample": f"one full step ({'+'.join('nv=%d' % v for v in wl['nvs'])} matvecs) "
                                      f"of {args.config} at full size per timed step, single-threaded C oracle"},
           "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)


def main():
    # keep stdout for the single JSON line: library / NCCL chatter goes to stderr
    json_fd = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(os.dup(2), "w")
    emit = lambda obj: os.write(json_fd, (json.dumps(obj) + "\n").encode())
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="no clocks / e2e / cpu (for ncu runs)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    wl = WORKLOADS[args.config]
    if args.impl == "reference":
        return run_reference(args, wl, emit)

    import torch
    import torch.distributed as dist
    import paper_2109_05451_b200 as pkg
    from h2gen import make_xy, SEED
    pkg.load_library()
    ws, rk, lr = dist_env()
    P = ws
    torch.cuda.set_device(lr)
    dev = torch.device("cuda", lr)
    if P > 1:
        dist.init_process_group("nccl", device_id=dev)
    t_gen = time.perf_counter()
    want_cpu = (P == 1 and rk == 0 and not args.no_cpu_baseline and not args.profile_only)
    tree, st, hglob, kw, (r0, r1) = build_problem(wl, P, rk, with_global=want_cpu)
    t_gen = time.perf_counter() - t_gen
    nccl_id = None
    if P > 1:
        from paper_2109_05451_b200.operator import broadcast_nccl_id
        nccl_id = broadcast_nccl_id(dev)
    nv_max = max(wl["nvs"])
    op = pkg.H2Operator(dtype=wl["dtype"], nv_max=nv_max, nccl_id=nccl_id, **kw)
    n_local = int(kw["n_local"])
    perm_local = tree.perm[r0:r1]
    tdt = torch.float64 if wl["dtype"] == "f64" else torch.float32
    X = {nv: torch.from_numpy(make_xy(perm_local, nv, SEED)).to(dev, tdt) for nv in wl["nvs"]}
    Y = {nv: torch.zeros(nv, n_local, dtype=tdt, device=dev) for nv in wl["nvs"]}
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if P > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def step():
        for nv in wl["nvs"]:
            op.matvec(X[nv], Y[nv], 1.0, 0.0, stream)

    for _ in range(args.warmup):
        step()
    barrier()
    # ---- timed region (device time, CUDA events on the launching stream)
    op.set_profiling(True)
    op.phase_times()                       # reset
    clocks = ClockSampler(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ else lr)
    per_nv_ms = {nv: 0.0 for nv in wl["nvs"]}
    per_nv_ph = {nv: {} for nv in wl["nvs"]}
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in wl["nvs"]] for _ in range(args.steps)]
    with (clocks if not args.profile_only else _Null()):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(args.steps):
            for i, nv in enumerate(wl["nvs"]):
                ev[s][i][0].record(stream)
                op.matvec(X[nv], Y[nv], 1.0, 0.0, stream)
                ev[s][i][1].record(stream)
        e1.record(stream)
        barrier()
    total_ms = e0.elapsed_time(e1)
    for s in range(args.steps):
        for i, nv in enumerate(wl["nvs"]):
            per_nv_ms[nv] += ev[s][i][0].elapsed_time(ev[s][i][1])
    phases, ncalls = op.phase_times()
    op.set_profiling(False)
    # per-nv phase times: one extra profiled pass per nv (same kernels; side streams serialized
    # so each phase's CUDA events bracket only its own launches)
    for nv in wl["nvs"]:
        op.set_profiling(True)
        for _ in range(3):
            op.matvec(X[nv], Y[nv], 1.0, 0.0, stream)
        per_nv_ph[nv], _ = op.phase_times()
        op.set_profiling(False)
    # max over ranks
    t = torch.tensor([total_ms] + [per_nv_ms[nv] for nv in wl["nvs"]], dtype=torch.float64, device=dev)
    if P > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t[0])
    for i, nv in enumerate(wl["nvs"]):
        per_nv_ms[nv] = float(t[i + 1]) / args.steps
    ms_step = total_ms / args.steps
    flops_rank = {nv: op.stats(nv)["flops"] for nv in wl["nvs"]}
    ft = torch.tensor([sum(flops_rank.values())] + [flops_rank[nv] for nv in wl["nvs"]], dtype=torch.float64, device=dev)
    if P > 1:
        dist.all_reduce(ft)
    flops_step = float(ft[0])
    value = flops_step / (ms_step * 1e-3) / 1e9
    launches = op.stats(1)["launches"]
    # ---- e2e through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e and not args.profile_only:
        Xh = {nv: torch.from_numpy(make_xy(perm_local, nv, SEED)).to(tdt).pin_memory() for nv in wl["nvs"]}
        Yh = {nv: torch.zeros(nv, n_local, dtype=tdt).pin_memory() for nv in wl["nvs"]}
        for nv in wl["nvs"]:
            op.matvec_host(Xh[nv], Yh[nv], 1.0, 0.0, stream)
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            for nv in wl["nvs"]:
                op.matvec_host(Xh[nv], Yh[nv], 1.0, 0.0, stream)
        b.record(stream)
        barrier()
        te = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
        if P > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te[0]) / args.steps
        esz = 8 if wl["dtype"] == "f64" else 4
        e2e = {"value": flops_step / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": sum(n_local * nv * esz for nv in wl["nvs"]),
               "d2h_bytes_per_step": sum(n_local * nv * esz for nv in wl["nvs"])}
    # ---- roofline of the dominant kernel (largest phase time over the step)
    hbm, hbm_src = peaks()
    step_ph = {k: sum(per_nv_ph[nv].get(k, 0.0) for nv in wl["nvs"]) for k in pkg.PHASES}
    # phases launched by the same kernel (the coupling rows of the tree levels and of the leaf
    # level are two k_rows<WRITE> launches) are one kernel for the roofline
    kof = pkg._binding.KERNEL_OF_PHASE
    groups = {}
    for k in pkg.PHASES:
        groups.setdefault(kof.get(k, k), []).append(k)
    dom_k = max(groups, key=lambda g: sum(step_ph[k] for k in groups[g]))
    dom_phases = groups[dom_k]
    dom = "+".join(dom_phases)
    bytes_dom = sum(op.phase_stats(nv)[0][k] for nv in wl["nvs"] for k in dom_phases)
    ms_dom = sum(step_ph[k] for k in dom_phases)
    achieved = bytes_dom / (ms_dom * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        if tr.get("config") == args.config and dom in tr.get("phases", {}):
            traffic = tr["phases"][dom]
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": dom_k,
                "phase": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "peak_source": hbm_src,
                "algorithmic_bytes_per_step": bytes_dom, "ms_per_step": ms_dom}
    # FP64 phases whose flops outlast their bytes at the measured peaks (nv = 64) are bounded by the
    # FP64 tensor pipe: report them against the measured cuBLAS DGEMM rate instead
    flops_dom = sum(op.phase_stats(nv)[1][k] for nv in wl["nvs"] for k in dom_phases)
    f64_tf, f64_src = fp64_peak()
    if wl["dtype"] == "f64" and flops_dom / (f64_tf * 1e12) > bytes_dom / (hbm * 1e9):
        ach_tf = flops_dom / (ms_dom * 1e-3) / 1e12
        roofline.update({"bound": "tensor", "achieved": ach_tf, "peak": f64_tf, "unit": "TFLOP/s",
                         "frac": ach_tf / f64_tf, "peak_source": f64_src,
                         "algorithmic_flops_per_step": flops_dom, "hbm_frac": achieved / hbm})
    # ---- CPU oracle beside it (rank 0, N=1 only): one full step, single thread
    cpu = None
    if want_cpu:
        import oracle
        prep = oracle.prepare(hglob)
        Xc = {nv: X[nv].double().cpu().numpy() for nv in wl["nvs"]}
        t0 = time.perf_counter()
        for nv in wl["nvs"]:
            oracle.matvec(hglob, Xc[nv], 1.0, 0.0, None, prepared=prep)
        sec = time.perf_counter() - t0
        cpu = {"value": flops_step / sec / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
               "sample": f"one full step ({'+'.join('nv=%d' % v for v in wl['nvs'])} matvecs) of "
                         f"{args.config} at full size, single-threaded C oracle, {sec:.1f} s"}
    if rk == 0:
        cfg = {"workload": f"{args.config}: {wl['desc']}", "N_global": int(tree.N), "N_per_gpu": n_local,
               "nvs": list(wl["nvs"]), "parallelism": f"block-rows x{P}" if P > 1 else "single GPU",
               "l2": "inputs larger than L2 (operator %.2f GB streamed per matvec; L2 126 MB)"
                     % (op.stats(1)["bytes"] / 1e9),
               "timing": "CUDA events on the launching stream, barrier+sync both sides, max over ranks",
               "gen_seconds": round(t_gen, 1)}
        out = {"metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": P, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": wl["dtype"], "data": "synthetic",
               "config": cfg,
               "per_nv": {str(nv): {"ms_per_matvec": per_nv_ms[nv],
                                    "gflops": float(ft[i + 1]) / (per_nv_ms[nv] * 1e-3) / 1e9,
                                    "gflops_per_gpu": float(ft[i + 1]) / (per_nv_ms[nv] * 1e-3) / 1e9 / P,
                                    "phases_ms": {k: round(v, 5) for k, v in per_nv_ph[nv].items()}}
                          for i, nv in enumerate(wl["nvs"])},
               "roofline": roofline,
               "path_bandwidth": {str(nv): {"algorithmic_bytes": op.stats(nv)["bytes"],
                                            "GB_s": op.stats(nv)["bytes"] / (per_nv_ms[nv] * 1e-3) / 1e9,
                                            "frac_of_hbm": op.stats(nv)["bytes"] / (per_nv_ms[nv] * 1e-3) / 1e9 / hbm}
                                  for nv in wl["nvs"]},
               "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": launches * len(wl["nvs"]) * args.steps,
               "clocks": clocks.summary() if not args.profile_only else None}
        emit(out)
    op.close()
    if P > 1:
        dist.barrier()
        dist.destroy_process_group()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass


if __name__ == "__main__":
    main()
