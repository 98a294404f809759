"""Benchmark: fine-DOF/s of the localized gamblet setup + subband solve (fp64).

Workload (BASELINE.json configs[2], "Single GPU"): q = 10 (N = 4^10 =
1,048,576 interior nodes under the reference's node convention), log-uniform
contrast-1e4 checkerboard coefficient (PCG64 seed 0), Gaussian nodal load
(seed 1), localized gamblets with uniform radius 3, reference tight mode
(epsilon = 1e-13, c_tol = 1e-6).  A "step" is one full fast_solve: setup of
every level (psi^(k), A^(k), B^(k), R, D, spectral estimates) plus all
subband solves and the reassembly of u.

  value  device-resident inputs (M, A as CSR in HBM, g in HBM), u left in HBM
  e2e    the public API gb.fast_solve with host scipy M, A and host load,
         host->device uploads and the device->host copy of u inside the step

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
        N > 1 (one process per GPU via torch.distributed.run, NCCL): BASELINE
        configs[3] (q = 12, 16.8 M DOFs) split spatially into N row strips --
        gamblet_dist.fast_solve_dist: per-rank strips of every level operator,
        neighbour halo exchanges, distributed PCG (strong scaling).  Configs 0
        and 4 run N replicas.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "c0": dict(q=5, coeff="example1", exact=True),
    "c1": dict(q=7, coeff="example1"),
    "c2": dict(q=10, coeff="checker"),
    "c3": dict(q=12, coeff="checker"),
    "c4": dict(q=7, coeff="example3d", d=3),
}
RHO3 = 2
EPS, RHO, CTOL = 1e-13, 3, 1e-6
METRIC = "fine-DOF/s for gamblet setup+solve (fp64)"
# CPU sample of configs 1-3: the oracle's complete tight-mode pipeline on a
# 2^CPU_WINDOW_Q x 2^CPU_WINDOW_Q block of the config's own instance
CPU_WINDOW_Q = 7
CPU_WINDOW_Q3 = 3


def instance_seeds(rank):
    """(coefficient seed, load seed) of the problem instance a rank solves:
    rank 0 is BASELINE's config (S_a = 0, S_g = 1); rank r solves the
    independent instance (2r, 2r + 1) of the same family."""
    return 2 * rank, 2 * rank + 1


def build_inputs(q, coeff, rank=0):
    import paper_1503_03467_b200 as gb
    grid = gb.build_grid(q)
    sa, sg = instance_seeds(rank)
    if coeff == "example1":
        c = gb.coefficient_example1(grid)
        g = gb.example_load(grid)
    else:
        c = gb.coefficient_checkerboard(grid, 1e4, sa)
        g = np.random.default_rng(sg).standard_normal(grid.num_nodes)
    M = gb.assemble_mass(grid)
    A = gb.assemble_stiffness(grid, c)
    load = gb.assemble_load(grid, g, mass=M)
    return grid, M, A, load, gb.build_hierarchy(grid)


def window_inputs(q, coeff, m, index):
    """Block `index` (row-major over the (2^q / 2^m)^2 disjoint blocks) of the
    config's own q-instance: its coefficient cells and nodal load restricted
    to a 2^m x 2^m node window with Dirichlet conditions on the window edge
    (the same coefficient statistics, patch sizes and localization radii)."""
    import paper_1503_03467_b200 as gb
    grid = gb.build_grid(q)
    if coeff == "example1":
        c = gb.coefficient_example1(grid).as_cell_grid()
        g = gb.example_load(grid).reshape(grid.n, grid.n)
    else:
        sa, sg = instance_seeds(0)
        c = gb.coefficient_checkerboard(grid, 1e4, sa).as_cell_grid()
        g = np.random.default_rng(sg).standard_normal(grid.num_nodes).reshape(grid.n, grid.n)
    w = 1 << m
    nb = grid.n // w
    bi, bj = divmod(int(index) % (nb * nb), nb)
    gw = gb.build_grid(m)
    cw = gb.CoefficientField(gw, c[bi * w:bi * w + w + 1, bj * w:bj * w + w + 1].ravel().copy())
    M = gb.assemble_mass(gw)
    A = gb.assemble_stiffness(gw, cw)
    load = gb.assemble_load(gw, g[bi * w:(bi + 1) * w, bj * w:(bj + 1) * w].ravel().copy(),
                            mass=M)
    return M, A, load, (bi, bj)


def window_order(q, m):
    """A fixed pseudo-random visiting order of the disjoint windows."""
    nb = (1 << q) >> m
    return np.random.default_rng(12345).permutation(nb * nb)


def cpu_oracle_sample(q, coeff, threads, index=0):
    """The CPU oracle (numpy/scipy restatement of the reference, tight mode,
    direct patch solves) over one window of the config's own instance:
    (fine-DOF/s, seconds, window)."""
    from threadpoolctl import threadpool_limits
    from oracle import gamblets_oracle as O
    m = min(q, CPU_WINDOW_Q)
    M, A, load, win = window_inputs(q, coeff, m, index)
    with threadpool_limits(threads):
        t0 = time.perf_counter()
        O.fast_solve(M, A, load.g_nodal, m, EPS, uniform_rho=RHO)
        dt = time.perf_counter() - t0
    return 4 ** m / dt, dt, win


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.proc = None
        self.path = Path(f"/tmp/gb_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        self.path.unlink(missing_ok=True)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


def fp64_peak_tflops():
    """Measured FP64 peak on this GPU: max of the DFMA and DMMA probes."""
    import torch
    from paper_1503_03467_b200 import _native as nat, device as dv
    sink = dv.empty(1)
    best = {}
    for kind, name in ((0, "dfma"), (1, "dmma")):
        iters = 4000
        nat.call("gb_fp64_peak_probe", kind, 200, dv.ptr(sink), dv.stream())
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        nat.call("gb_fp64_peak_probe", kind, iters, dv.ptr(sink), dv.stream())
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        if kind == 0:
            flops = 148 * 8 * 256 * iters * 8 * 8 * 2.0
        else:
            flops = 148 * 8 * 8 * iters * 8 * 256 * 2.0   # warps * iters * 8 mma * 256 FMA
        best[name] = flops / (ms * 1e-3) / 1e12
    return best


def kernel_timings(levels, q):
    """The finest level's Krylov operator, and the finest correction-patch
    launch re-timed in isolation (CUDA events on the launching stream) on the
    level's own B^(q) and a nonzero G block."""
    import torch
    from paper_1503_03467_b200 import _native as nat, device as dv, gamblet_fast as gf
    lv = levels[q]
    op = lv._op
    s = dv.stream()
    B = lv.raw("subband")
    if B is None:  # lean transform (q >= 12): the subband box is not retained
        return {"op": op, "corr": None}
    rho = min(3, B.L - 1)
    Dt = dv.empty(B.L * B.L * dv.box_slots(rho, 3))
    st = dv.zeros(2, torch.int64)
    G = dv.to_dev(np.ones(B.rows * dv.box_slots(B.w, 1)))  # nonzero right-hand sides
    ws, nb = gf._correction_ws(B.L, rho, 0, B.L)
    args = (B.L, B.w, dv.ptr(B.vals), dv.ptr(lv.raw("subband_scale")), B.w, dv.ptr(G), rho,
            dv.ptr(Dt), dv.ptr(st), dv.ptr(ws), nb, s)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nat.call("gb_correction_patches_v2", *args)
    torch.cuda.synchronize()
    a.record()
    nat.call("gb_correction_patches_v2", *args)
    b.record()
    torch.cuda.synchronize()
    return {"op": op, "corr": {"ms": a.elapsed_time(b), "flops": gf._patch_flops(B.L, rho, 3)}}


def ncu_traffic(config, q, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`
    from this config's committed ncu --set full capture
    (profiles/r02_ncu_traffic.json), or None when it was not captured."""
    f = ROOT / "profiles" / "r02_ncu_traffic.json"
    if not f.exists():
        return None
    return json.loads(f.read_text()).get(f"{config}:q{q}:{kernel}")


def workload_config(name, q, world):
    """The `config` object both arms print (identical for the same run)."""
    cfg = CONFIGS[name]
    N = 4 ** q
    if cfg.get("exact"):
        return {"workload": f"{name}: q={q}, N={N} fine DOFs, exact (global) gamblets, "
                            "tight mode tol 1e-14", "q": q, "fine_dofs": N,
                "parallelism": "single GPU" if world == 1 else f"{world} replicas"}
    if cfg.get("d") == 3:
        N = 8 ** q
        return {"workload": f"{name}: 3-D unit cube, q={q} ({1 << q}^3 = {N} fine DOFs), "
                            f"Q1 trilinear 27-point, example coefficient, localized gamblets "
                            f"rho={RHO3}, tight mode eps={EPS}",
                "q": q, "d": 3, "fine_dofs": N, "rho": RHO3, "epsilon": EPS,
                "parallelism": "single GPU" if world == 1 else f"{world} replicas",
                "l2": "working set > 126 MB L2 (operators tens of GB), no flush needed"}
    return {"workload": f"{name}: q={q}, N={N} fine DOFs, {cfg['coeff']}, "
                        f"localized gamblets rho={RHO}, tight mode eps={EPS}",
            "q": q, "fine_dofs": N, "rho": RHO, "epsilon": EPS,
            "parallelism": (f"{world} independent seeded instances, one per GPU "
                            "(weak scaling, no data-path collective)")
                           if world > 1 else "single GPU",
            "l2": "working set > 126 MB L2 (operators ~GBs), no flush needed",
            "lean": bool(q >= 12)}


def reduce_max(value, world, device=None):
    """Max over ranks of a per-rank time (the step is as slow as its slowest
    rank); identity on one process."""
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(dofs_per_rank, world, ms):
    """Weak scaling over independent instances: every rank solves N fine DOFs;
    the job rate is world * N per (max-over-ranks) step time."""
    return world * dofs_per_rank / (ms * 1e-3)


def run_exact(args, rank, world, local_rank):
    """BASELINE configs[0]: exact (global) gamblets, q=5, through the public
    exact_solve with host inputs in tight mode (tol 1e-14); each step is one
    complete call (uploads, dense sweep, reassembly, u download)."""
    import torch
    import paper_1503_03467_b200 as gb
    from paper_1503_03467_b200 import _native as nat, device as dv
    torch.cuda.set_device(local_rank)
    cfg = CONFIGS[args.config]
    q = args.q or cfg["q"]
    N = 4 ** q
    grid, M, A, load, tree = build_inputs(q, cfg["coeff"], rank)

    def step():
        sol, _ = gb.exact_solve(M, A, load, tree, tol_mass=1e-14, tol_subband=1e-14)
        return sol.u

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = nat.query("gb_launch_count")
    seg0 = torch.cuda.memory_stats().get("segment.all.allocated", 0)
    dv.Traffic.reset()
    with ClockSampler(local_rank) as clk:
        ts = []
        for _ in range(args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            step()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
    launches = nat.query("gb_launch_count") - launches0
    # cudaMalloc calls inside the timed region (each stalls every stream)
    new_segments = torch.cuda.memory_stats().get("segment.all.allocated", 0) - seg0
    ms = reduce_max(float(np.median(ts)), world, "cuda")
    if rank != 0:
        return None
    value = whole_job_rate(N, world, ms)
    return {
        "metric": METRIC, "value": round(value, 1), "unit": "fine-DOF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generators: example1 coefficient and load)",
        "config": workload_config(args.config, q, world),
        "e2e": {"value": round(value, 1), "unit": "fine-DOF/s", "ms_per_step": round(ms, 3),
                "h2d_bytes_per_step": int(dv.Traffic.h2d / max(1, args.steps)),
                "d2h_bytes_per_step": int(dv.Traffic.d2h / max(1, args.steps))},
        "gpu_launches": int(launches), "roofline": None,
        "note": "launch/latency-bound dense path (SURVEY 8(d): ~6.4 GFlop total); "
                "value is measured through the public call with host inputs",
        "clocks": clk.summary(), "step_ms": [round(t, 2) for t in ts],
    }


def build_inputs_3d(q, rank=0):
    from paper_1503_03467_b200 import gamblet_3d as g3
    grid = g3.build_grid_3d(q)
    _, sg = instance_seeds(rank)
    c = g3.coefficient_example_3d(grid)
    M = g3.assemble_mass_3d(grid)
    A = g3.assemble_stiffness_3d(grid, c)
    g = g3.gaussian_load_3d(grid, sg)
    return grid, M, A, g


def run_3d(args, rank, world, local_rank):
    """BASELINE configs[4]: 3-D unit cube 128^3 (q = 7), Q1 trilinear,
    example coefficient, Gaussian nodal load (seed 1), rho = 2, tight mode.
    value: M, A as device boxes and g in HBM; e2e: fast_solve_3d with host
    scipy CSR M, A and host g, uploads and the u download inside the step."""
    import torch
    from paper_1503_03467_b200 import _native as nat, device as dv, gamblet_3d as g3
    torch.cuda.set_device(local_rank)
    q = args.q or CONFIGS[args.config]["q"]
    N = 8 ** q
    grid, M, A, g = build_inputs_3d(q, rank)
    Md, Ad = g3.box3_from_csr(M, 1 << q), g3.box3_from_csr(A, 1 << q)
    gd = dv.to_dev(g)

    def step():
        return g3.fast_solve_3d(Md, Ad, gd, q, EPS, uniform_rho=RHO3)

    for _ in range(args.warmup):
        res = step()
        res = None
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    launches0 = nat.query("gb_launch_count")
    dv.Prof.reset(enabled=True)  # CUDA-event spans of the phases, live in the timed steps
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record()
        for _ in range(args.steps):
            res = None
            res = step()
            torch.cuda.synchronize()
        ev1.record()
        torch.cuda.synchronize()
    launches = nat.query("gb_launch_count") - launches0
    phase_ms = {k: v / args.steps for k, v in dv.Prof.times_ms().items()}
    dv.Prof.reset(enabled=False)
    ms = reduce_max(ev0.elapsed_time(ev1) / args.steps, world, "cuda")
    iters = dict(res.iterations)
    res = None
    e2e_ms = []
    dv.Traffic.reset()
    for _ in range(max(1, min(args.steps, 2))):
        res = None
        torch.cuda.synchronize()
        dv.Traffic.reset()
        t0 = time.perf_counter()
        res = g3.fast_solve_3d(M, A, g, q, EPS, uniform_rho=RHO3)
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        h2d, d2h = dv.Traffic.h2d, dv.Traffic.d2h
    e2e = reduce_max(float(np.median(e2e_ms)), world, "cuda")
    if rank != 0:
        return None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sample_3d(q, os.cpu_count() or 1, 0)
    # roofline of the dominant kernel: the correction patches of every level
    # (k3_correction_patches, batched blocked Cholesky on the FP64 tensor
    # cores), algorithmic flops sum over patches of m^3/3 + 2 m^2 with
    # m = 7 x the clipped ball, over the phase's live CUDA-event span
    roof = None
    corr_ms = phase_ms.get("3d_correction_patches")
    if corr_ms:
        flops = 0.0
        for k in range(q, 1, -1):
            Lp = 1 << (k - 1)
            rho = min(RHO3, Lp - 1)
            ext = np.minimum(np.arange(Lp), rho) + np.minimum(Lp - 1 - np.arange(Lp), rho) + 1
            m = 7.0 * np.multiply.outer(np.multiply.outer(ext, ext), ext).ravel()
            flops += float((m ** 3 / 3.0 + 2.0 * m * m).sum())
        fp64 = fp64_peak_tflops()
        peak = max(fp64.values())
        ach = flops / (corr_ms * 1e-3) / 1e12
        roof = {"kernel": "k3_correction_patches (all levels: batched blocked Cholesky of the "
                          "875 x 875 patch matrices, DMMA m8n8k4 trailing updates)",
                "bound": "tensor", "achieved": round(ach, 3), "peak": round(peak, 3),
                "unit": "TFLOP/s", "frac": round(ach / peak, 4), "traffic": None,
                "peak_source": "FP64 tensor-core (DMMA) probe measured in-run; "
                               "MEASURED_PEAKS.json has no fp64 figure",
                "flops_per_step": flops, "ms_per_step": round(corr_ms, 2),
                "timing": "CUDA events on the launching stream around the phase in every "
                          "timed step"}
    return {
        "metric": METRIC, "value": round(whole_job_rate(N, world, ms), 1), "unit": "fine-DOF/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (3-D example coefficient of BASELINE configs[4], Gaussian nodal "
                "load seed 1)",
        "config": workload_config(args.config, q, world),
        "e2e": {"value": round(whole_job_rate(N, world, e2e), 1), "unit": "fine-DOF/s",
                "ms_per_step": round(e2e, 3), "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches), "roofline": roof,
        "phases_ms": {k: round(v, 2) for k, v in sorted(phase_ms.items(), key=lambda x: -x[1])},
        "cpu_baseline": cpu, "clocks": clk.summary(),
        "krylov_iterations": {str(k): v for k, v in iters.items()},
    }


def cpu_sample_3d(q, threads, index):
    """The 3-D restatement (oracle/gamblets_oracle_nd.py, tight mode, rho=2)
    on one 2^m-per-axis window of the config's own instance."""
    from threadpoolctl import threadpool_limits
    from oracle import gamblets_oracle_nd as ND
    from paper_1503_03467_b200 import gamblet_3d as g3
    m = min(q, CPU_WINDOW_Q3)
    grid = g3.build_grid_3d(q)
    c = g3.coefficient_example_3d(grid).reshape((grid.n + 1,) * 3)
    g = g3.gaussian_load_3d(grid, 1).reshape((grid.n,) * 3)
    w = 1 << m
    nb = grid.n // w
    bi, bj, bk = np.unravel_index(int(index) % (nb ** 3), (nb,) * 3)
    gw = g3.build_grid_3d(m)
    cw = c[bi * w:bi * w + w + 1, bj * w:bj * w + w + 1, bk * w:bk * w + w + 1].ravel().copy()
    M = g3.assemble_mass_3d(gw)
    A = g3.assemble_stiffness_3d(gw, cw)
    gv = g[bi * w:(bi + 1) * w, bj * w:(bj + 1) * w, bk * w:(bk + 1) * w].ravel().copy()
    with threadpool_limits(threads):
        t0 = time.perf_counter()
        ND.fast_solve(M, A, gv, m, 3, EPS, uniform_rho=RHO3)
        dt = time.perf_counter() - t0
    return {"value": round(8 ** m / dt, 2), "unit": "fine-DOF/s", "cores": threads,
            "kind": "port",
            "sample": f"oracle/gamblets_oracle_nd.fast_solve (d=3, tight mode, rho={RHO3}) on "
                      f"window {(int(bi), int(bj), int(bk))} ({w}^3 nodes = {8 ** m} DOFs) of "
                      f"this config's own q={q} instance, {dt:.1f} s"}


def run_ours(args, rank, world, local_rank):
    import torch
    import paper_1503_03467_b200 as gb
    from paper_1503_03467_b200 import _native as nat, device as dv, gamblet_fast as gf

    torch.cuda.set_device(local_rank)
    cfg = CONFIGS[args.config]
    q = args.q or cfg["q"]
    coeff = cfg["coeff"]
    N = 4 ** q
    grid, M, A, load, tree = build_inputs(q, coeff, rank)
    sched = gb.make_schedule(EPS, q, uniform_rho=RHO)

    # device-resident inputs for the `value` leg
    Md = dv.DeviceCSR.from_scipy(M)
    Ad = dv.DeviceCSR.from_scipy(A)
    gd = dv.to_dev(load.g_nodal)

    # q >= 12: the memory-bounded transform (same arithmetic; level operators
    # released once consumed) -- 16.8 M DOFs do not fit otherwise
    lean = q >= 12

    def step_device():
        levels, parts, U1, counter = gf._fast_solve_device(Md, Ad, gd, tree, sched, lean=lean)
        return levels, parts, counter

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for i in range(args.warmup):
        step_device()
        if i == 0 and not lean:
            # grow the caching allocator once to the step's high-water mark
            # (+50% against fragmentation): later steps make no cudaMalloc,
            # which would stall every stream of the level engine (the lean
            # q >= 12 runs use expandable segments instead)
            dv.reserve(1.5 * torch.cuda.max_memory_allocated())
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    dv.Prof.reset(enabled=True)
    # live timing of the dominant kernel inside the timed steps: the finest
    # level's engine records CUDA events on its own stream around every
    # dual-vector phase-1 launch (k_symb_apply_ws<2>) of every step
    gf.ENGINE_TIMING = {"n": 3 * 4 ** (q - 1), "cap": 512, "ms": []}
    launches0 = nat.query("gb_launch_count")
    seg0 = torch.cuda.memory_stats().get("segment.all.allocated", 0)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record()
        marks = []
        levels = parts = counter = None
        for _ in range(args.steps):
            # drop the previous step's outputs first: holding two steps' level
            # operators at once overflows the reserved pool (cudaMalloc stalls)
            levels = parts = counter = None
            levels, parts, counter = step_device()
            marks.append(torch.cuda.Event(enable_timing=True))
            marks[-1].record()
            # a step is one complete solve: the host waits for it (as a caller
            # reading its results would) before the next one is enqueued
            torch.cuda.synchronize()
        ev1.record()
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches = nat.query("gb_launch_count") - launches0
    # cudaMalloc calls inside the timed region (each stalls every stream)
    new_segments = torch.cuda.memory_stats().get("segment.all.allocated", 0) - seg0
    ms = ev0.elapsed_time(ev1) / args.steps
    step_ms = [round(ev0.elapsed_time(marks[0]), 1)] + [
        round(a.elapsed_time(b_), 1) for a, b_ in zip(marks, marks[1:])]
    engine_ms = list(gf.ENGINE_TIMING.get("ms", []))
    gf.ENGINE_TIMING = None
    phase_ms = {k: v / args.steps for k, v in dv.Prof.times_ms().items()}
    phase_flops = {k: v / args.steps for k, v in dv.Prof.flops.items()}
    phase_bytes = {k: v / args.steps for k, v in dv.Prof.bytes.items()}
    phase_counts = {k: v // args.steps for k, v in dv.Prof.counts().items()}
    # timeline of the last step: (start, end) ms of every phase instance,
    # relative to the first event recorded in that step
    evs = dv.Prof.events[-(len(dv.Prof.events) // args.steps):]
    t0 = evs[0][1]
    timeline = [(lbl, round(t0.elapsed_time(a), 2), round(t0.elapsed_time(b_), 2))
                for lbl, a, b_ in evs]
    dv.Prof.reset(enabled=False)
    ms = reduce_max(ms, world, "cuda")
    value = whole_job_rate(N, world, ms)
    iters = {k: v for k, v in counter.iterations.items()}

    # e2e through the public API with host buffers
    e2e_ms = []
    h2d = d2h = 0
    levels = parts = None  # the device leg's last outputs are not needed any more
    Md = Ad = gd = None    # nor its device-resident inputs (3.9 GB at q=12)
    res = None
    # one untimed call first: the allocator adapts to the host-input pattern
    res = gb.fast_solve(M, A, load, tree, EPS, uniform_rho=RHO, c_tol=CTOL, lean=lean)
    res = None
    for i in range(max(1, args.steps)):
        res = None  # as in the device leg: one solve's operators live at a time
        torch.cuda.synchronize()
        barrier()
        dv.Traffic.reset()
        t0 = time.perf_counter()
        res = gb.fast_solve(M, A, load, tree, EPS, uniform_rho=RHO, c_tol=CTOL, lean=lean)
        u = res.solution.u  # host copy made inside the call
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        h2d, d2h = dv.Traffic.h2d, dv.Traffic.d2h
    e2e = reduce_max(float(np.median(e2e_ms)), world, "cuda")
    levels = res.levels  # device-backed level objects of the last solve
    del res

    if rank != 0:
        return None

    # isolated timing of the dominant kernels on the last solve's finest level
    kern = kernel_timings(levels, q)

    # repeat solves on the stored transform ("subsequent
    # solves"): K loads one call at a time vs one batched call (subband PCGs
    # two at a time through the dual-vector SpMV), host loads in, u out
    rep = None
    if args.repeat_solves > 0 and not lean:
        sched = res_sched = gb.make_schedule(EPS, q, uniform_rho=RHO)
        rng = np.random.default_rng(99)
        loads = [gb.assemble_load(grid, rng.standard_normal(grid.num_nodes), mass=M)
                 for _ in range(args.repeat_solves)]
        gb.solve_with_transform(levels, loads[:2], tree, res_sched)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for ld in loads:
            gb.solve_with_transform(levels, ld, tree, sched)
        torch.cuda.synchronize()
        t_single = (time.perf_counter() - t0) / len(loads)
        t0 = time.perf_counter()
        gb.solve_with_transform(levels, loads, tree, sched)
        torch.cuda.synchronize()
        t_batch = (time.perf_counter() - t0) / len(loads)
        rep = {"loads": len(loads), "ms_per_load_single": round(t_single * 1e3, 3),
               "ms_per_load_batched": round(t_batch * 1e3, 3),
               "fine_dofs_per_s_batched": round(N / t_batch, 1),
               "fine_dofs_per_s_single": round(N / t_single, 1),
               "note": "solve_with_transform on the stored transform, host loads "
                       "(g uploaded, u downloaded) inside the timing; wall clock with a "
                       "device synchronize on both sides"}

    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs")
    hbm_src = ("MEASURED_PEAKS.json hbm_gbs (measured copy)" if hbm_peak
               else "fallback 6650 GB/s of B200_PROFILING.md")
    hbm_peak = hbm_peak or 6650.0
    fp64 = fp64_peak_tflops()
    fp64_peak = max(fp64.values())

    # roofline of the dominant kernel: k_symb_apply_ws<2>, the finest level's
    # dual-vector pass (subband PCG + Lanczos halves) of the symmetric band
    # S B S SpMV, timed live inside the timed steps on the engine's stream.
    # Algorithmic bytes per launch: the stored upper 3x3 blocks once, plus x
    # read and y written for each of the two vectors
    op = kern["op"]
    dual_bytes = op.matrix_bytes + 4 * 8 * op.n
    roof = None
    if engine_ms:
        em = np.sort(np.asarray(engine_ms, dtype=float))
        dual_ms = float(em.mean())
        achieved = dual_bytes / (dual_ms * 1e-3) / 1e9
        # the engine's stream shares the GPU with the FP64 setup kernels of the
        # main stream for the first part of a step (by design: the step is
        # shorter); the fastest half of the launches ran after the setup ended
        excl_ms = float(em[: max(1, len(em) // 2)].mean())
        excl = dual_bytes / (excl_ms * 1e-3) / 1e9
        roof = {"kernel": "k_symb_apply_ws<2> (finest-level S B S dual-vector pass: symmetric "
                          "band, upper 3x3 blocks streamed once by bulk copies, lower half "
                          "applied by scatter; PCG + Lanczos vectors)",
                "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak,
                "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                "traffic": ncu_traffic(args.config, q, "k_symb_apply_ws<2>"),
                "peak_source": hbm_src, "bytes_per_launch": int(dual_bytes),
                "ms_per_launch": round(dual_ms, 4), "launches_timed": len(engine_ms),
                "not_overlapped": {"ms_per_launch": round(excl_ms, 4),
                                   "achieved": round(excl, 1),
                                   "frac": round(excl / hbm_peak, 4),
                                   "launches": int(max(1, len(em) // 2)),
                                   "what": "the fastest half of the same in-step launches: "
                                           "those issued after the main stream's FP64 setup "
                                           "kernels, which share the SMs with the earlier "
                                           "ones, had finished"},
                "timing": "CUDA events on the level engine's stream around every dual launch "
                          "of the finest level in every timed step"}
    cp = kern["corr"]
    fp = None if cp is None else {
        "kernel": "k_correction_patches_v3 (finest level, left-looking tiled DMMA Cholesky, "
                  "L streamed through an L2-resident scratch)",
        "bound": "fp64", "achieved": round(cp["flops"] / (cp["ms"] * 1e-3) / 1e12, 3),
        "peak": round(fp64_peak, 3), "unit": "TFLOP/s",
        "frac": round(cp["flops"] / (cp["ms"] * 1e-3) / 1e12 / fp64_peak, 4),
        "peak_source": "measured in-run (max of DFMA/DMMA probes; MEASURED_PEAKS.json "
                       "has no fp64 figure)",
        "ms_per_launch": round(cp["ms"], 3), "flops_per_launch": cp["flops"],
        "timing": "isolated re-launch after the timed region on the finest level's own B and "
                  "its G block (CUDA events, same stream)"}

    # aggregate step roofline: sum over phases of
    # max(algorithmic flops / fp64 peak, algorithmic bytes / HBM peak), against
    # the measured step time (phases on different streams overlap)
    agg_phases = {}
    roof_ms = 0.0
    for lbl in sorted(set(phase_flops) | set(phase_bytes)):
        f_ms = phase_flops.get(lbl, 0) / (fp64_peak * 1e12) * 1e3
        b_ms = phase_bytes.get(lbl, 0) / (hbm_peak * 1e9) * 1e3
        roof_ms += max(f_ms, b_ms)
        agg_phases[lbl] = {"roof_ms": round(max(f_ms, b_ms), 3),
                           "bound": "fp64" if f_ms > b_ms else "hbm",
                           "measured_ms": round(phase_ms.get(lbl, 0.0), 3),
                           "gflop": round(phase_flops.get(lbl, 0) / 1e9, 2),
                           "gbytes": round(phase_bytes.get(lbl, 0) / 1e9, 3)}
    aggregate = {"roofline_ms": round(roof_ms, 3), "step_ms": round(ms, 3),
                 "frac": round(roof_ms / ms, 4),
                 "dofs_per_s_at_roofline": round(N / (roof_ms * 1e-3), 1),
                 "note": "per-phase measured_ms are CUDA-event spans per step on the "
                         "launching stream; spans on the level-engine streams overlap the "
                         "main stream",
                 "phases": agg_phases}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, dt, win = cpu_oracle_sample(q, coeff, threads, index=int(window_order(q, min(q, CPU_WINDOW_Q))[0]))
        m = min(q, CPU_WINDOW_Q)
        cpu = {"value": round(v, 2), "unit": "fine-DOF/s", "cores": threads, "kind": "port",
               "sample": f"oracle/gamblets_oracle.fast_solve (tight mode) over window {win} "
                         f"({1 << m}x{1 << m} nodes = {4 ** m} DOFs) of this config's own "
                         f"q={q} instance, {dt:.1f} s"}

    clocks = clk.summary()
    out = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "fine-DOF/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded reference generators: checkerboard contrast 1e4 seed 0, "
                "Gaussian nodal load seed 1)",
        "config": workload_config(args.config, q, world),
        "e2e": {"value": round(whole_job_rate(N, world, e2e), 1), "unit": "fine-DOF/s",
                "ms_per_step": round(e2e, 3), "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches),
        "gpu_launches_per_step": int(launches // max(1, args.steps)),
        "allocator_segments_timed": int(new_segments),
        "roofline": roof,
        "roofline_fp64": fp,
        "roofline_aggregate": aggregate,
        "repeat_solves": rep,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "step_ms": step_ms,
        "phases_ms": {k: round(v, 3) for k, v in sorted(phase_ms.items(), key=lambda x: -x[1])},
        "phase_launch_groups": phase_counts,
        "timeline_last_step_ms": timeline if args.timeline else None,
        "fp64_peak_tflops": {k: round(v, 2) for k, v in fp64.items()},
        "subband_iterations": iters.get("line8"),
        "spectral_iterations": [
            {"n": d["n"], "power": d["power"], "lanczos": d["lanczos"], "outer": d["outer"]}
            if "lanczos" in d else {"n": d["n"], "power": d["power"], "inner_cg": d["inner"]}
            for d in gf._SPECTRAL_LOG[-(q - 1):]],
    }
    return out


def run_dist(args, rank, world, local_rank):
    """N > 1: the spatially partitioned solve (gamblet_dist.fast_solve_dist)
    of ONE instance -- BASELINE configs[3] unless --config says otherwise --
    over `world` ranks: strong scaling, value = N fine DOFs / step time (max
    over ranks, device-timed).  value: M, A device-assembled boxes (9 values
    per row, replicated) and g in HBM; e2e: the host coefficient cells and the
    host nodal load in (on-device Q1 assembly, grid_fem.assemble_*(device=True):
    bitwise the reference's CSR values), u back on the host, on every rank --
    no rank builds the 150 M-entry scipy matrices of q = 12."""
    import torch
    import torch.distributed as dist
    import paper_1503_03467_b200 as gb
    from paper_1503_03467_b200 import _native as nat, device as dv, gamblet_dist as gd
    torch.cuda.set_device(local_rank)
    name = args.config if args.config_given else "c3"
    cfg = CONFIGS[name]
    q = args.q or cfg["q"]
    N = 4 ** q
    comm = gb.TorchComm()
    if rank == 0:
        print(f"[bench] partitioned run: world {world}, backend {comm.backend}, q={q}; "
              f"one {comm.backend} communicator over ranks 0..{world - 1}"
              + (" (NCCL_DEBUG=INFO prints its channels)" if comm.backend == "nccl" else ""),
              file=sys.stderr)
    # the one instance every rank shares (rank-0 seeds of BASELINE's config)
    grid = gb.build_grid(q)
    tree = gb.build_hierarchy(grid)
    if cfg["coeff"] == "example1":
        c = gb.coefficient_example1(grid)
        g_host = gb.example_load(grid)
    else:
        sa, sg = instance_seeds(0)
        c = gb.coefficient_checkerboard(grid, 1e4, sa)
        g_host = np.random.default_rng(sg).standard_normal(grid.num_nodes)
    Mb = gb.assemble_mass(grid, device=True)
    Ab = gb.assemble_stiffness(grid, c, device=True)
    gd_dev = dv.to_dev(g_host)

    def step():
        return gd.fast_solve_dist(comm, Mb, Ab, gd_dev, tree, EPS, uniform_rho=RHO)

    for _ in range(args.warmup):
        res = step()
        res = None
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    gd.DIST_TIMING = {"n": 3 * 4 ** (q - 1), "cap": 64, "ms": []}
    launches0 = nat.query("gb_launch_count")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record()
        for _ in range(args.steps):
            res = None
            res = step()
            torch.cuda.synchronize()
        ev1.record()
        torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    launches = nat.query("gb_launch_count") - launches0
    timing, gd.DIST_TIMING = gd.DIST_TIMING, None
    ms = reduce_max(ev0.elapsed_time(ev1) / args.steps, world, "cuda")
    peak = reduce_max(res.peak_bytes, world, "cuda")
    halo = reduce_max(res.halo_bytes, world, "cuda")
    its, lams, first_rep, passes = res.iterations, res.lambdas, res.first_replicated, \
        res.krylov_passes
    res = None
    # e2e: host inputs in, u on the host out, every step
    e2e_ms = []
    for _ in range(max(1, min(args.steps, 3))):
        torch.cuda.synchronize()
        dist.barrier()
        dv.Traffic.reset()
        t0 = time.perf_counter()
        M2 = gb.assemble_mass(grid, device=True)
        A2 = gb.assemble_stiffness(grid, c, device=True)   # uploads the cell values
        r2 = gd.fast_solve_dist(comm, M2, A2, g_host, tree, EPS, uniform_rho=RHO)
        u = dv.to_host(r2.u)
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        h2d, d2h = dv.Traffic.h2d, dv.Traffic.d2h
        r2 = M2 = A2 = None
    e2e = reduce_max(float(np.median(e2e_ms)), world, "cuda")
    if rank != 0:
        return None
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs") or 6650.0
    roof = None
    if timing.get("ms"):
        dual_ms = float(np.mean(timing["ms"]))
        nbytes = timing["matrix_bytes"] + timing["vector_bytes"]
        ach = nbytes / (dual_ms * 1e-3) / 1e9
        roof = {"kernel": "k_symb_apply_ws<2> on the rank's tile rows (finest level, strip of "
                          "the symmetric band S B S, PCG + spectral vectors)",
                "bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(ach / hbm_peak, 4), "traffic": None,
                "bytes_per_launch": int(nbytes), "ms_per_launch": round(dual_ms, 4),
                "launches_timed": len(timing["ms"]),
                "timing": "CUDA events on rank 0's stream around its first 64 dual launches "
                          "of the finest level in every timed step (per GPU)"}
    # the same configuration on ONE GPU (the N = 1 bench line is configs[2]):
    # the committed single-GPU measurement of this config, for a like-for-like
    # parallel efficiency
    single = None
    sf = ROOT / "profiles" / f"r02_bench_{name}.json"
    if sf.exists() and not args.q:
        sd = json.loads(sf.read_text())
        single = {"value": sd["value"], "unit": sd["unit"], "ms_per_step": sd["ms_per_step"],
                  "source": f"profiles/{sf.name} (bench.py --config {name} on one B200)"}
    cfgo = workload_config(name, q, world)
    cfgo["parallelism"] = (f"spatial row strips over {world} GPUs: levels with >= "
                           f"{gd.min_distributed_rows(world)} parent rows distributed (halo "
                           f"exchange + all-reduce over NCCL), coarser levels replicated with "
                           f"column strips of psi; first replicated level {first_rep}")
    return {
        "metric": METRIC, "value": round(N / (ms * 1e-3), 1), "unit": "fine-DOF/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded reference generators, one instance shared by all ranks)",
        "config": cfgo,
        "e2e": {"value": round(N / (e2e * 1e-3), 1), "unit": "fine-DOF/s",
                "ms_per_step": round(e2e, 3), "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": int(launches), "roofline": roof, "cpu_baseline": None,
        "clocks": clk.summary(),
        "single_gpu_same_config": single,
        "per_rank_peak_bytes": int(peak), "per_rank_halo_bytes_per_step": int(halo),
        "subband_iterations": {str(k): v for k, v in sorted(its.items())},
        "krylov_passes": {str(k): list(v) for k, v in passes.items()},
        "lambdas": {str(k): list(v) for k, v in sorted(lams.items())},
    }


def run_reference(args, rank, world):
    """Reference arm: the CPU oracle port (numpy/scipy restatement of the
    reference, tight mode, direct patch solves; the reference itself is pure
    Python and cannot travel to the GPU box), all host threads.

    Config 0: the complete q=5 exact sweep every step.  Configs 1-3: every
    step is the oracle's complete pipeline (transform + subband solves) on one
    2^7 x 2^7-node window of the config's OWN instance (its coefficient cells
    and load; steps visit different windows in a fixed order), and the rate
    is window DOFs / time.  The oracle's cost per DOF is level-size
    independent (O(patch) gathers), so the window rate is the instance's
    rate; the reference itself is super-linear (O(N) per patch extraction),
    so this over-states the reference at q=10."""
    if rank != 0:
        return None
    from threadpoolctl import threadpool_limits
    from oracle import gamblets_oracle as O
    cfg = CONFIGS[args.config]
    q = args.q or cfg["q"]
    threads = os.cpu_count() or 1
    if cfg.get("d") == 3:  # config 4: windows of the 3-D instance, 3-D restatement
        times, wins = [], []
        m = min(q, CPU_WINDOW_Q3)
        for i in range(args.warmup + args.steps):
            r = cpu_sample_3d(q, threads, i)
            if i >= args.warmup:
                times.append(8 ** m / r["value"])
                wins.append(r["sample"])
        dt = float(np.mean(times))
        value = 8 ** m / dt
        return {
            "impl": "reference", "metric": METRIC, "value": round(value, 2),
            "unit": "fine-DOF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt * 1e3, 1), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (same instance as the GPU arm)",
            "config": workload_config(args.config, q, world),
            "cpu_baseline": {"value": round(value, 2), "unit": "fine-DOF/s", "cores": threads,
                             "kind": "port",
                             "sample": f"oracle/gamblets_oracle_nd.fast_solve (d=3, the "
                                       f"reference has no 3-D) on one {1 << m}^3-node window "
                                       f"of the config's own q={q} instance per step"},
            "e2e": {"value": round(value, 2), "unit": "fine-DOF/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }
    if cfg.get("exact"):  # config 0: the whole q=5 exact sweep fits a CPU step
        grid, M, A, load, tree = build_inputs(q, cfg["coeff"])
        times = []
        with threadpool_limits(threads):
            for i in range(args.warmup + args.steps):
                t0 = time.perf_counter()
                O.exact_solve(M, A, load.b, q)
                if i >= args.warmup:
                    times.append(time.perf_counter() - t0)
        dofs = 4 ** q
        sample = (f"oracle/gamblets_oracle.exact_solve (dense direct restatement of the "
                  f"reference's exact sweep), the full q={q} config every step")
    else:
        m = min(q, CPU_WINDOW_Q)
        order = window_order(q, m)
        times, wins = [], []
        for i in range(args.warmup + args.steps):
            _, dt, win = cpu_oracle_sample(q, cfg["coeff"], threads, index=int(order[i % len(order)]))
            if i >= args.warmup:
                times.append(dt)
                wins.append(win)
        dofs = 4 ** m
        sample = (f"oracle/gamblets_oracle.fast_solve (tight mode, uniform rho={RHO}) on one "
                  f"{1 << m}x{1 << m}-node window ({dofs} DOFs) of this config's own q={q} "
                  f"instance per step (coefficient cells and load of the window, Dirichlet on "
                  f"its edge); {len(set(wins))} distinct windows timed")
    dt = float(np.mean(times))
    value = dofs / dt
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 2),
        "unit": "fine-DOF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 1), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded reference generators, same instance as the GPU arm)",
        "config": workload_config(args.config, q, world),
        "cpu_baseline": {"value": round(value, 2), "unit": "fine-DOF/s", "cores": threads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 2), "unit": "fine-DOF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS))
    ap.add_argument("--q", type=int, default=None, help="override the config's q")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--timeline", action="store_true")
    ap.add_argument("--repeat-solves", type=int, default=4,
                    help="loads of the repeat-solve leg (0: skip)")
    args = ap.parse_args()
    args.config_given = args.config is not None
    world = int(os.environ.get("WORLD_SIZE", "1"))
    # N = 1: configs[2]; N > 1: configs[3] split over the GPUs (both arms)
    args.config = args.config or ("c3" if world > 1 else "c2")
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if (args.q or CONFIGS[args.config]["q"]) >= 12:
        # 16.8 M DOFs on one GPU: expandable allocator segments, and a third
        # Krylov worker so queued levels release their psi^(k) sooner
        os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
        os.environ.setdefault("GB_SPECTRAL_WORKERS", "3")
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            # GB_DIST_BACKEND=gloo: functional runs of the N > 1 path on fewer
            # GPUs than ranks (ranks share devices, rows staged through the
            # host) -- never a measurement
            backend = os.environ.get("GB_DIST_BACKEND", "nccl")
            if backend != "nccl":
                local_rank = local_rank % max(1, torch.cuda.device_count())
            torch.cuda.set_device(local_rank)
            torch.distributed.init_process_group(backend)
        cfg = CONFIGS[args.config]
        runner = run_exact if cfg.get("exact") else run_3d if cfg.get("d") == 3 else run_ours
        if world > 1 and runner is run_ours:
            runner = run_dist
        out = runner(args, rank, world, local_rank)
        if world > 1:
            import torch
            torch.distributed.destroy_process_group()
    if out is not None:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
