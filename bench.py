#!/usr/bin/env python
"""bench.py — H² matvec throughput on B200 (driver contract; DESIGN.md §"Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config suite]

A workload LEG is one BASELINE.json config in one precision with its vector counts; one STEP of a
leg is one pass of the whole hot path (upsweep, coupling, downsweep, dense near field, epilogue)
for every nv of the leg, on inputs already resident in HBM.

--config suite (default) times
  * the PRIMARY leg cfg2 (BASELINE configs[1]: 2D exp kernel, 1M points per GPU, nv = 1 and 16,
    FP64; weak scaling at N > 1): `value`, `ms_per_step`, `per_nv`, `roofline`, `e2e`;
  * cfg3 (configs[2]: 3D Gaussian, 2M points, k = 64, nv = 64, FP64; STRONG scaling: the same 2M
    points split over the N GPUs) and cfg1 (configs[0]: N = 4096, latency, warm / cold L2) as
    extra legs under `per_config`, each with its own roofline, e2e and CPU baseline.
--config cfg2|cfg3|cfg3s|cfg4|cfg5|cfg1: that workload alone as the primary leg (cfg5 = FP64 and
    FP32 legs).
Timing: CUDA events on the launching stream, barrier + device sync on both sides, max over ranks;
the timed loop runs the product path (one CUDA graph per call, concurrent side stream); per-phase
times come from a separate profiled pass afterwards.  Rank 0 prints one JSON line.
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
# a workload name with ":sym" = the same workload on the symmetric-storage path (H2_SYMMETRIC,
# nv = 1 legs only: SURVEY.md §8(f) NEXT-2); ":f32" / ":f64" = one precision of a workload
SUITES = {
    "suite": (["cfg2"], ["cfg3", "cfg5:f32", "cfg2:sym", "cfg1"]),
    "cfg2sym": (["cfg2:sym"], []), "cfg4sym": (["cfg4:sym"], []),
    "cfg1": (["cfg1"], []), "cfg2": (["cfg2"], []), "cfg3": (["cfg3"], []), "cfg3s": (["cfg3s"], []),
    "cfg4": (["cfg4"], []), "cfg5": (["cfg5"], []), "cfg5f32": (["cfg5:f32"], []),
}
CPU_BUDGET_S = 12.0          # oracle seconds per leg for the cpu_baseline sample


# ------------------------------------------------------------------------------------------ helpers
def fp_peaks():
    """Measured peaks: HBM copy bandwidth (MEASURED_PEAKS.json), FP64 / FP32 GEMM rates (cuBLAS
    DGEMM / SGEMM 8192^3 measured on this pool's B200, profiles/peaks_b200_r01.json)."""
    out = {"hbm": (6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"), "f64": (40.0, "nominal FP64 40 TFLOP/s"),
           "f32": (80.0, "nominal FP32 80 TFLOP/s")}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            out["hbm"] = (float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)")
    except Exception:
        pass
    try:
        with open(os.path.join(ROOT, "profiles", "peaks_b200_r01.json")) as f:
            pk = json.load(f)
        out["f64"] = (float(pk["gemm_float64_tflops"]), "measured cuBLAS DGEMM 8192^3 (profiles/peaks_b200_r01.json)")
        out["f32"] = (float(pk["gemm_float32_tflops"]), "measured cuBLAS SGEMM 8192^3 (profiles/peaks_b200_r01.json)")
    except Exception:
        pass
    return out


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

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
            self.f.seek(0)
            self.lines = self.f.read().splitlines()
        self.f.close()
        os.unlink(self.f.name)


def clock_summary(samplers):
    lines = [ln for s in samplers for ln in s.lines]
    if not any(s.proc for s in samplers):
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
    sm, smax, reasons = [], None, set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for line in lines:
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
    busy = [s for s in sm if smax and s > 0.5 * smax] or sm
    return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": smax,
            "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def legs_of(name):
    """[(config, dtype, nvs)] of one workload (cfg5: one leg per precision; "name:sym": the
    symmetric-storage path, nv = 1 only)."""
    from h2gen.configs import CONFIGS
    base, _, opt = name.partition(":")
    c = CONFIGS[base]
    if opt == "sym":
        return [(name, dt, (1,)) for dt in c["dtypes"]]
    if opt in ("f32", "f64"):                 # one precision of a multi-precision workload
        return [(name, opt, tuple(c["nvs"]))]
    return [(name, dt, tuple(c["nvs"])) for dt in c["dtypes"]]


def leg_key(leg):
    name, dt, nvs = leg
    return f"{name}/{dt}/nv={'+'.join(map(str, nvs))}"


def base_name(name):
    return name.partition(":")[0]


def config_dict(args, P, legs_primary, legs_extra, N_global, n_local):
    from h2gen.configs import CONFIGS
    prim = base_name(legs_primary[0][0])
    scal = CONFIGS[prim]["scaling"]
    return {"workload": "; ".join(f"{leg_key(lg)}: {CONFIGS[base_name(lg[0])]['desc']}" for lg in legs_primary),
            "extra_legs": [leg_key(lg) for lg in legs_extra],
            "N_global": N_global, "N_per_gpu": n_local,
            "parallelism": f"block rows x{P} ({scal} scaling)" if P > 1 else "single GPU",
            "l2": "inputs larger than L2 (operators of 5-40 GB streamed per matvec; L2 126 MB); cfg1 (L2-resident) "
                  "reported warm and cold (256 MB scrub between reps)",
            "timing": "CUDA events on the launching stream, barrier+sync both sides, max over ranks; product path "
                      "(CUDA graph); phase split from a separate profiled pass"}


# ---------------------------------------------------------------------------------- problem setup
def build_leg_problem(name, P, rank, with_global):
    """(tree, host operator kwargs for this rank, (r0, r1), global H2Data or None)."""
    from h2gen.configs import build_structure
    from h2gen.h2data import build_h2
    from h2gen.shard import build_h2_shard
    tree, st, kern, c = build_structure(base_name(name), P)
    if with_global or P == 1:
        from paper_2109_05451_b200.operator import shard_arrays
        h = build_h2(tree, st, kern, c["p"])
        kw, rows = shard_arrays(h, rank, P)
        return tree, kw, rows, h, c
    kw, rows = build_h2_shard(tree, st, kern, c["p"], rank, P)
    return tree, kw, rows, None, c


def cast_kw(kw, dtype):
    if dtype == "f64":
        return kw
    kw = dict(kw)
    f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float32)
    for key in ("U_leaf", "V_leaf", "D"):
        kw[key] = f(kw[key])
    for key in ("E", "F", "S"):
        kw[key] = [f(a) for a in kw[key]]
    return kw


# ------------------------------------------------------------------------------ CPU oracle leg
def oracle_work(h, mask):
    """Scalar multiply-adds per vector the oracle performs with leaf mask `mask` (None = all):
    full upsweep, couplings / downsweep on the ancestors of the masked leaves, their dense rows.
    Used only to scale a sampled oracle time to the whole workload."""
    q = h.q
    rows = np.diff(np.asarray(h.leaf_ptr))
    need = [None] * (q + 1)
    need[q] = np.ones(1 << q, dtype=bool) if mask is None else np.asarray(mask, dtype=bool)
    for l in range(q - 1, -1, -1):
        need[l] = need[l + 1][0::2] | need[l + 1][1::2]
    k = h.ranks
    w = float(rows.sum()) * k[q] + sum(float(1 << l) * k[l] * k[l - 1] for l in range(1, q + 1))
    for l in range(q + 1):
        nb = np.diff(np.asarray(h.S_rowptr[l]))
        w += float(nb[need[l]].sum()) * k[l] * k[l]
        if l >= 1:
            w += float(need[l].sum()) * k[l] * k[l - 1]
    w += float(rows[need[q]].sum()) * k[q]
    drp = np.asarray(h.D_rowptr)
    trow = np.repeat(np.arange(1 << q), np.diff(drp))
    sel = need[q][trow]
    w += float((rows[trow[sel]] * rows[np.asarray(h.D_col)[sel]]).sum())
    return w


def oracle_mask(h, nvs, budget_s, cores):
    """Leaf sample sized for ~budget_s of oracle time (assumed ~2.5 GFLOP/s per core; the rate only
    sizes the sample, the reported value is measured)."""
    full = oracle_work(h, None) * 2.0 * sum(nvs)
    frac = min(1.0, budget_s * 2.5e9 * cores / max(full, 1.0))
    if frac >= 1.0:
        return None, 1.0
    rng = np.random.default_rng(12345)
    mask = rng.random(1 << h.q) < max(frac, 1.0 / (1 << h.q))
    return mask, oracle_work(h, mask) / oracle_work(h, None)


def time_oracle(h, Xs, nvs, mask, flops_model, frac):
    import oracle
    prep = oracle.prepare(h)
    t0 = time.perf_counter()
    for nv in nvs:
        oracle.matvec(h, Xs[nv], 1.0, 0.0, None, leaf_mask=mask, prepared=prep)
    sec = time.perf_counter() - t0
    return sec, flops_model * frac / sec / 1e9


def run_reference(args, emit):
    """--impl reference: the CPU oracle (oracle/, plain C FP64 + OpenMP over the host cores) on the
    primary legs of the same workload, rank 0 only; each step = every matvec of the legs on a
    bounded leaf sample sized so the whole --steps/--warmup run stays within a few minutes."""
    ws, rk, _ = dist_env()
    if rk != 0:
        return
    import oracle
    from h2gen import make_xy, SEED
    cores = oracle.set_threads(0)
    prim, extra = SUITES[args.config]
    legs = [lg for nm in prim for lg in legs_of(nm)]
    parts, flops_step, sample = [], 0.0, []
    # the oracle's rate is timed on the one-GPU workload: its GFLOP/s does not depend on the global
    # size, and building a P-GPU weak-scaled operator on the host (8x cfg2 = tens of GB) would not
    # fit the reference arm's minutes; the config reported is the P-GPU one (structure only)
    for name, dt, nvs in legs:
        _, _, _, h, c = build_leg_problem(name, 1, 0, True)
        hh = h if dt == "f64" else h.astype(np.float32).astype(np.float64)
        Xs = {nv: make_xy(h.perm, nv, SEED) for nv in nvs}
        fl = sum(h.flops(nv) for nv in nvs)
        budget = 150.0 / (args.steps + args.warmup) / len(legs)
        mask, frac = oracle_mask(h, nvs, budget, cores)
        parts.append((hh, Xs, nvs, mask, fl, frac))
        flops_step += fl
        sample.append(f"{leg_key((name, dt, nvs))}: {frac * 100:.1f}% of the oracle work (leaf sample, full upsweep)"
                      + (f" of the one-GPU workload (rate; the {ws}-GPU global operator is not built)" if ws > 1 else ""))

    def step():
        return sum(time_oracle(hh, Xs, nvs, mask, fl, frac)[0] / frac for hh, Xs, nvs, mask, fl, frac in parts)
    for _ in range(args.warmup):
        step()
    t = [step() for _ in range(args.steps)]          # each step's time scaled to the full step
    sec = sum(t) / len(t)
    val = flops_step / sec / 1e9
    from h2gen.configs import CONFIGS
    P = ws
    n_first = int(parts[0][0].N)
    n_rank0 = n_first
    if P > 1:
        # per-GPU rows of rank 0 = its branch at the C-level (the same rows the GPU arm reports)
        from h2gen.configs import build_structure
        tree_p = build_structure(base_name(legs[0][0]), P)[0]
        C = P.bit_length() - 1
        lp = np.asarray(tree_p.leaf_ptr)
        n_first = int(tree_p.N)
        n_rank0 = int(lp[1 << (tree_p.q - C)])
    legs_x = [lg for nm in extra for lg in legs_of(nm) if not (P > 1 and lg[0].endswith(":sym"))]
    ours_cfg = config_dict(args, ws, legs, legs_x, n_first, n_rank0)
    out = {"metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
           "scaling": CONFIGS[base_name(legs[0][0])]["scaling"], "vs_baseline": None, "dtype": legs[0][1], "data": "synthetic",
           "config": ours_cfg, "impl": "reference",
           "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                            "sample": "; ".join(sample) + "; time scaled by the work fraction"},
           "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)


# ------------------------------------------------------------------------------------ GPU legs
def run_leg(leg, args, P, rank, dev, pkg, torch, dist, want_cpu, samplers, latency=False):
    from h2gen import make_xy, SEED
    name, dtype, nvs = leg
    t_gen = time.perf_counter()
    tree, kw, (r0, r1), hglob, cfg = build_leg_problem(name, P, rank, want_cpu)
    t_gen = time.perf_counter() - t_gen
    nccl_id = None
    if P > 1:
        from paper_2109_05451_b200.operator import broadcast_nccl_id
        nccl_id = broadcast_nccl_id(dev)
    sym = name.endswith(":sym")
    kw = cast_kw(kw, dtype)
    if sym:                                   # H2_SYMMETRIC: U = V and E = F as one array each
        kw = dict(kw, V_leaf=kw["U_leaf"], F=kw["E"])
    op = pkg.H2Operator(dtype=dtype, nv_max=max(nvs), nccl_id=nccl_id, symmetric=sym, **kw)
    del kw
    n_local = int(op.n_local)
    perm_local = tree.perm[r0:r1]
    tdt = torch.float64 if dtype == "f64" else torch.float32
    esz = 8 if dtype == "f64" else 4
    X = {nv: torch.from_numpy(make_xy(perm_local, nv, SEED)).to(dev, tdt) for nv in nvs}
    Y = {nv: torch.zeros(nv, n_local, dtype=tdt, device=dev) for nv in nvs}
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if P > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        for nv in nvs:
            op.matvec(X[nv], Y[nv], 1.0, 0.0, stream)
    barrier()
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in nvs]
          for _ in range(args.steps)]
    scrub = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if latency else None
    cold = []
    gidx = torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ else dev.index
    sampler = ClockSampler(gidx) if not args.profile_only else None
    with (sampler if sampler else _Null()):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(args.steps):
            for i, nv in enumerate(nvs):
                ev[s][i][0].record(stream)
                op.matvec(X[nv], Y[nv], 1.0, 0.0, stream)
                ev[s][i][1].record(stream)
        e1.record(stream)
        barrier()
        if latency:                         # cold L2: a 256 MB scrub before every call
            for s in range(args.steps):
                for i, nv in enumerate(nvs):
                    scrub.add_(1)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    op.matvec(X[nv], Y[nv], 1.0, 0.0, stream)
                    b.record(stream)
                    cold.append((a, b))
            barrier()
    if sampler:
        samplers.append(sampler)
    per_nv_ms = [sum(ev[s][i][0].elapsed_time(ev[s][i][1]) for s in range(args.steps)) for i in range(len(nvs))]
    t = torch.tensor([e0.elapsed_time(e1)] + per_nv_ms, dtype=torch.float64, device=dev)
    if P > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t[0]) / args.steps
    per_nv_ms = {nv: float(t[i + 1]) / args.steps for i, nv in enumerate(nvs)}
    fl = torch.tensor([op.stats(nv)["flops"] for nv in nvs], dtype=torch.float64, device=dev)
    if P > 1:
        dist.all_reduce(fl)
    flops = {nv: float(fl[i]) for i, nv in enumerate(nvs)}
    flops_step = sum(flops.values())
    launches = op.stats(1)["launches"]
    # per-phase times: a separate profiled pass (side stream serialised; events between phases)
    per_nv_ph = {}
    for nv in nvs:
        op.set_profiling(True)
        op.phase_times()
        for _ in range(3):
            op.matvec(X[nv], Y[nv], 1.0, 0.0, stream)
        per_nv_ph[nv], _ = op.phase_times()
        op.set_profiling(False)
    # e2e through the public API with pinned host buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e and not args.profile_only:
        Xh = {nv: torch.from_numpy(make_xy(perm_local, nv, SEED)).to(tdt).pin_memory() for nv in nvs}
        Yh = {nv: torch.zeros(nv, n_local, dtype=tdt).pin_memory() for nv in nvs}
        for nv in nvs:
            op.matvec_host(Xh[nv], Yh[nv], 1.0, 0.0, stream)
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            for nv in nvs:
                op.matvec_host(Xh[nv], Yh[nv], 1.0, 0.0, stream)
        b.record(stream)
        barrier()
        te = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
        if P > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te[0]) / args.steps
        e2e = {"value": flops_step / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": sum(n_local * nv * esz for nv in nvs),
               "d2h_bytes_per_step": sum(n_local * nv * esz for nv in nvs)}
        del Xh, Yh
    # roofline of the leg's dominant kernel (largest summed phase time)
    pk = fp_peaks()
    kof = dict(pkg._binding.KERNEL_OF_PHASE)
    if dtype == "f64" and max(nvs) > 16 and not name.endswith(":sym"):   # the CTA-tile engine runs these legs
        kof.update({"up_leaf": "k_cta<leaf projection>", "up_transfer": "k_cta<upsweep levels>",
                    "coupling_diag": "k_cta<coupling rows>", "coupling_leaf": "k_cta<coupling rows>",
                    "coupling_offdiag": "k_cta<coupling rows, off-diagonal>", "down_transfer": "k_cta<downsweep levels>",
                    "leaf_u": "k_cta<leaves: expansion + dense + epilogue>", "dense": "k_cta<leaves: expansion + dense + epilogue>"})
    if dtype == "f32" and min(nvs) >= 5 and os.environ.get("H2_ENGINE") != "warp":   # tcgen05 engine
        kof.update({"coupling_diag": "k_umma<rows> (tcgen05)", "coupling_leaf": "k_umma<rows> (tcgen05)",
                    "coupling_offdiag": "k_umma<rows> (tcgen05)",
                    "leaf_u": "k_umma<leaf> (tcgen05; + leaf-level E rows)", "dense": "k_umma<leaf> (tcgen05; + leaf-level E rows)"})
    if name.endswith(":sym"):
        kof.update({"coupling_diag": "k_sym_rows", "coupling_leaf": "k_sym_rows", "leaf_u": "k_sym_leaf",
                    "dense": "k_sym_leaf"})
    step_ph = {k: sum(per_nv_ph[nv].get(k, 0.0) for nv in nvs) for k in pkg.PHASES}
    groups = {}
    for k in pkg.PHASES:
        groups.setdefault(kof.get(k, k), []).append(k)
    dom_k = max(groups, key=lambda g: sum(step_ph[k] for k in groups[g]))
    dom_phases = groups[dom_k]
    bytes_dom = sum(op.phase_stats(nv)[0][k] for nv in nvs for k in dom_phases)
    flops_dom = sum(op.phase_stats(nv)[1][k] for nv in nvs for k in dom_phases)
    ms_dom = sum(step_ph[k] for k in dom_phases)
    hbm, hbm_src = pk["hbm"]
    fpk, fpk_src = pk[dtype]
    gbs = bytes_dom / (ms_dom * 1e-3) / 1e9
    if flops_dom / (fpk * 1e12) > bytes_dom / (hbm * 1e9):
        tf = flops_dom / (ms_dom * 1e-3) / 1e12
        roof = {"bound": "tensor" if dtype == "f64" else "alu", "achieved": tf, "peak": fpk, "unit": "TFLOP/s",
                "frac": tf / fpk, "peak_source": fpk_src, "algorithmic_flops_per_step": flops_dom,
                "hbm_frac": gbs / hbm}
    else:
        roof = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                "peak_source": hbm_src}
    roof.update({"kernel": dom_k, "phase": "+".join(dom_phases), "algorithmic_bytes_per_step": bytes_dom,
                 "ms_per_step": ms_dom, "traffic": ncu_traffic(leg_key(leg), "+".join(dom_phases))})
    out = {"leg": leg_key(leg), "desc": cfg["desc"], "dtype": dtype, "N_global": int(tree.N), "N_per_gpu": n_local,
           "scaling": cfg["scaling"], "ms_per_step": ms_step, "gflops": flops_step / (ms_step * 1e-3) / 1e9,
           "gflops_per_gpu": flops_step / (ms_step * 1e-3) / 1e9 / P, "flops_step": flops_step,
           "per_nv": {str(nv): {"ms_per_matvec": per_nv_ms[nv],
                                "gflops": flops[nv] / (per_nv_ms[nv] * 1e-3) / 1e9,
                                "gflops_per_gpu": flops[nv] / (per_nv_ms[nv] * 1e-3) / 1e9 / P,
                                "path_frac_of_hbm": op.stats(nv)["bytes"] / (per_nv_ms[nv] * 1e-3) / 1e9 / hbm,
                                "phases_ms": {k: round(v, 5) for k, v in per_nv_ph[nv].items()}} for nv in nvs},
           "roofline": roof, "e2e": e2e, "launches_per_matvec": launches,
           "gpu_launches": launches * len(nvs) * args.steps, "gen_seconds": round(t_gen, 1)}
    if latency:
        cold_us = sorted(a.elapsed_time(b) * 1e3 for a, b in cold)
        warm_us = sorted(ev[s][i][0].elapsed_time(ev[s][i][1]) * 1e3 for s in range(args.steps) for i in range(len(nvs)))
        out["latency_us"] = {"warm_median": warm_us[len(warm_us) // 2], "warm_min": warm_us[0],
                             "cold_median": cold_us[len(cold_us) // 2], "cold_min": cold_us[0],
                             "launches_per_matvec": launches}
    # CPU oracle beside it (rank 0, N = 1): bounded leaf sample on all host cores
    if want_cpu and hglob is not None:
        import oracle
        cores = oracle.set_threads(0)
        hh = hglob if dtype == "f64" else hglob.astype(np.float32).astype(np.float64)
        Xc = {nv: X[nv].double().cpu().numpy() for nv in nvs}
        mask, frac = oracle_mask(hglob, nvs, CPU_BUDGET_S, cores)
        sec, val = time_oracle(hh, Xc, nvs, mask, flops_step, frac)
        out["cpu_baseline"] = {"value": val, "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                               "sample": f"{leg_key(leg)}: {frac * 100:.1f}% of the oracle work per step (random "
                                         f"leaf sample, full upsweep), {sec:.1f} s, OpenMP on {cores} host threads; "
                                         "scaled by the work fraction"}
    op.close()
    del X, Y, op, hglob
    torch.cuda.empty_cache()
    return out


def ncu_traffic(key, phases):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        return tr.get(key, {}).get(phases)
    except Exception:
        return None


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
    ap.add_argument("--config", default="suite", choices=sorted(SUITES))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="primary legs only")
    ap.add_argument("--profile-only", action="store_true", help="no clocks / e2e / cpu (for ncu runs)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args, emit)

    import torch
    import torch.distributed as dist
    import paper_2109_05451_b200 as pkg
    pkg.load_library()
    ws, rk, lr = dist_env()
    P = ws
    torch.cuda.set_device(lr)
    dev = torch.device("cuda", lr)
    if P > 1:
        dist.init_process_group("nccl", device_id=dev)
    prim, extra = SUITES[args.config]
    if args.no_extra or args.profile_only:
        extra = []
    legs_p = [lg for nm in prim for lg in legs_of(nm)]
    legs_x = [lg for nm in extra for lg in legs_of(nm) if not (P > 1 and lg[0].endswith(":sym"))]   # one rank only
    want_cpu = (P == 1 and rk == 0 and not args.no_cpu_baseline and not args.profile_only)
    samplers = []
    res_p = [run_leg(lg, args, P, rk, dev, pkg, torch, dist, want_cpu, samplers, latency=(lg[0] == "cfg1"))
             for lg in legs_p]
    res_x = [run_leg(lg, args, P, rk, dev, pkg, torch, dist, want_cpu, samplers, latency=(lg[0] == "cfg1"))
             for lg in legs_x]
    if rk == 0:
        ms_step = sum(r["ms_per_step"] for r in res_p)
        flops_step = sum(r["flops_step"] for r in res_p)
        value = flops_step / (ms_step * 1e-3) / 1e9
        dom = max(res_p, key=lambda r: r["roofline"]["ms_per_step"])
        per_nv = {}
        for r in res_p:
            for nv, d in r["per_nv"].items():
                per_nv[nv if len(res_p) == 1 else f"{r['leg']}"] = d
        e2e = None
        if all(r["e2e"] for r in res_p):
            e_ms = sum(r["e2e"]["ms_per_step"] for r in res_p)
            e2e = {"value": flops_step / (e_ms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": e_ms,
                   "h2d_bytes_per_step": sum(r["e2e"]["h2d_bytes_per_step"] for r in res_p),
                   "d2h_bytes_per_step": sum(r["e2e"]["d2h_bytes_per_step"] for r in res_p)}
        cpu = None
        if all("cpu_baseline" in r for r in res_p):
            cpu_s = sum(r["flops_step"] / (r["cpu_baseline"]["value"] * 1e9) for r in res_p)
            cpu = {"value": flops_step / cpu_s / 1e9, "unit": "GFLOP/s", "cores": res_p[0]["cpu_baseline"]["cores"],
                   "kind": "oracle", "sample": "; ".join(r["cpu_baseline"]["sample"] for r in res_p)}
        from h2gen.configs import CONFIGS
        out = {"metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": P, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
               "scaling": CONFIGS[base_name(legs_p[0][0])]["scaling"], "vs_baseline": None, "dtype": legs_p[0][1],
               "data": "synthetic",
               "config": config_dict(args, P, legs_p, legs_x, res_p[0]["N_global"], res_p[0]["N_per_gpu"]),
               "per_nv": per_nv, "roofline": dom["roofline"], "e2e": e2e, "cpu_baseline": cpu,
               "gpu_launches": sum(r["gpu_launches"] for r in res_p),
               "clocks": clock_summary(samplers) if not args.profile_only else None,
               "per_config": {r["leg"]: r for r in res_p + res_x}}
        emit(out)
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
