#!/usr/bin/env python
"""bench.py -- GN-step solves/s of the B200 Woodbury-MINRES solver (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl gnw|reference]

Workload (N=1 line): BASELINE.json configs[1] = C2, the configuration the metric is quoted
on: 512x512 unit square x 2 triangles (N = 524288 cells, K = 787456 edges), synthetic
J = U diag(s) V^T (m = 256), alpha sweep {1e-4, 1e-3, 1e-2, 1e-1, 1}, MINRES to 1e-8, FP64.
One STEP = one full GN-step solve = the reference's t_norm (inversion.cpp:242-271):
build_woodbury_preconditioner (H = S^-1 J^T by V-cycles, C = I + J H / alpha, chol C)
+ assemble_gn_rhs + MINRES; step k uses alpha = sweep[k % 5].  Inputs (J: 1.07 GB, H: 1.07 GB
per solve) are far larger than the 126 MB L2, so no L2 flush is needed between steps.

* value  -- device-resident inputs (torch CUDA tensors, device-pointer mode), timed with CUDA
            events on the library's stream; whole-job throughput (N replicas, max over ranks).
* e2e    -- the same solves through the C-ABI with HOST buffers (pinned): J, m, m_ref, g, g_obs
            copied H2D every step inside the timed region, x copied back D2H (gnw_set_jacobian +
            gnw_gn_step_solve: the reference's GN step, inversion.cpp:244-265).  Step k+1's
            J (1.07 GB) is staged with gnw_prefetch_jacobian during step k's MINRES (copy stream);
            step 0 copies its own J, so every step's input transfer is inside the timed region.
* roofline -- the dominant per-iteration kernel measured in isolation with CUDA events
            (gnw_profile_kernel), algorithmic bytes per SURVEY.md 8(d); peak = MEASURED_PEAKS.json.
* cpu_baseline -- the unmodified reference (oracle/_ref) on this host, 1 core (the reference is
            single-threaded): a bounded sample of the same C2 solve extrapolated to one full
            solve with the reference's own iteration count (tests/golden/c2_reference.json).

Multi-GPU: C2 does not shard (replicas only) -- N independent replicas, one
process per GPU, scaling "weak".  `--impl reference` runs the reference arm (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GN-step solves/s (MINRES+Woodbury-MG to 1e-8, FP64); % of HBM roofline"
UNIT = "GN-step solves/s"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks_dist(x: float, ws: int) -> float:
    """Max of a per-rank device time over all ranks (NCCL on GPUs, gloo on CPU)."""
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_throughput(elapsed_local: float, steps: int, ws: int) -> tuple[float, float]:
    """Whole-job solves/s of N independent replicas: N * steps / (max over ranks of the time)."""
    el = max_over_ranks_dist(elapsed_local, ws)
    return ws * steps / el, el


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.marks = []

    def mark(self):
        if not self.marks:
            time.sleep(0.25)  # let the sampler produce lines before the region starts
        self.marks.append(len(self.lines))

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.lines
        if len(self.marks) >= 2:  # the timed region (plus one sample either side)
            lines = self.lines[max(0, self.marks[0] - 1):self.marks[1] + 1]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def c2_reference_record():
    path = os.path.join(ROOT, "tests", "golden", "c2_reference.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


# CUDA kernel behind each gnw_profile_kernel name
KERNEL_NAMES = {"row_gemv": "k_row_gemv", "saddle": "k_saddle", "saddle_fused": "k_saddle (q from the finish sweep)",
                "finish_prec": "k_finish_prec", "finish_fused": "k_finish_prec (+ q = J^T t')",
                "vcycle": "V-cycle", "update": "k_minres_update", "col_sweep": "k_col_sweep (q = J^T t')",
                "finish_lean": "k_finish_prec (w = B q)"}


def cpu_sample(cfg, inp, alpha, iterations, k_cols=16, k_rows=16, k_iters=10, label="C2"):
    """Bounded sample of the reference on this host, extrapolated to one full GN-step solve."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import orc  # CPU baseline leg only

    o = orc.Oracle("reference" if orc.available("reference") else "restatement")
    p = orc.Problem.mixed(o, inp.mesh, orc.AmgOpts.make(coarse_threshold=cfg.coarse_threshold))
    if o.kind != "reference":
        raise RuntimeError("reference library oracle/_ref/libertinv_ref.so missing")
    t0 = time.time()
    s = p.sample_gnstep(inp.J, alpha, k_cols, k_rows, k_iters)
    wall = time.time() - t0
    t_est = s["t_col"] * cfg.m + s["t_row"] * cfg.m + s["t_chol"] + s["t_minres0"] + s["t_iter"] * iterations
    sample = (f"reference (oracle/_ref, -O3 -DNDEBUG) on {label} alpha={alpha:g}: {k_cols} H columns (V-cycles), "
              f"{k_rows} capacitance rows (matmul), full {cfg.m}x{cfg.m} Cholesky, MINRES runs of {k_iters} and "
              f"{2 * k_iters} iterations (per-iteration cost and minres's fixed start-up separated) "
              f"({wall:.1f} s of CPU); per-unit times x (m={cfg.m} columns, m rows, {iterations} iterations) "
              f"-> t_norm = {t_est:.1f} s")
    return 1.0 / t_est, t_est, s, sample, o.kind


def host_info() -> dict:
    """The host the CPU legs ran on: logical CPUs, CPU model, memory."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    mem = None
    try:
        import psutil
        mem = round(psutil.virtual_memory().total / 2**30, 1)
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "mem_gib": mem}


def reference_iterations(config: str) -> dict:
    """Per-alpha MINRES iteration counts of the reference's OWN full solves at tol 1e-8 on the
    seeded bundle of `config` (committed fixtures, tests/golden/).  Empty when none exist."""
    if config == "C2":
        rec = c2_reference_record()
        return {r["alpha"]: r["iterations"] for r in rec["runs"]} if rec else {}
    return {}


def _ref_worker(job):
    """One reference process (spawned, so the reference library is loaded by a fresh
    interpreter): loads the shared bundle, runs the bounded sample or a full solve."""
    path, n, m, thr, alpha, iters, kc, kr, ki, label, full = job
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import orc  # CPU baseline leg only
    from paper_2209_02815_b200 import workload as W

    d = np.load(path)
    inp = _Inputs()
    inp.mesh, inp.J, inp.dm, inp.dg = W.unit_square_mesh(n), d["J"], d["dm"], d["dg"]
    cfg = _Cfg(n=n, m=m, coarse_threshold=thr)
    if full:  # the whole t_norm measured: set_jacobian + assemble_gn_rhs + minres (inversion.cpp:242-271)
        o = orc.Oracle("reference")
        p = orc.Problem.mixed(o, inp.mesh, orc.AmgOpts.make(coarse_threshold=thr))
        t0 = time.time()
        p.set_jacobian(inp.J, alpha)
        b = p.assemble_rhs(inp.dm, np.zeros(p.N), inp.dg, np.zeros(m))
        x, rep = p.minres(b, tol=1e-8)
        t = time.time() - t0
        return t, (f"reference (oracle/_ref, -O3 -DNDEBUG) on {label} alpha={alpha:g}: one full GN-step solve "
                   f"measured ({rep['iterations']} MINRES iterations, t_norm {t:.3f} s)"), o.kind
    v, t_est, s, sample, kind = cpu_sample(cfg, inp, alpha, iters, k_cols=kc, k_rows=kr, k_iters=ki, label=label)
    return t_est, sample, kind


def ref_processes(job_bytes: float):
    """Independent reference processes the host can run at once: one per logical CPU, capped
    by memory (a C2 sample holds J, a J-sized H and the hierarchy: ~3 GB).  Returns
    (processes, memory_capped)."""
    n = os.cpu_count() or 1
    capped = False
    try:
        import psutil
        by_mem = max(1, int(0.6 * psutil.virtual_memory().available / job_bytes))
        capped = by_mem < n
        n = min(n, by_mem)
    except Exception:
        pass
    return max(1, n), capped


def cpu_sample_parallel(path, cfg, alpha, iterations, procs, k_cols, k_rows, k_iters, label, full):
    """The reference is single-threaded: to use every host core the same job runs as
    `procs` independent spawned processes at once (one solve each); throughput is the sum of
    their solves/s, each measured (or extrapolated from its own timings) under the shared load."""
    import multiprocessing as mp

    job = (path, cfg.n, cfg.m, cfg.coarse_threshold, alpha, iterations, k_cols, k_rows, k_iters, label, full)
    with mp.get_context("spawn").Pool(procs) as pool:
        res = pool.map(_ref_worker, [job] * procs)
    ts = [r[0] for r in res]
    value = sum(1.0 / t for t in ts)
    sample = (f"{procs} concurrent single-threaded reference processes, each: {res[0][1]}; "
              f"per-process t_norm {min(ts):.2f}-{max(ts):.2f} s; value = sum of 1 / t_norm")
    return value, ts, sample, res[0][2]


def full_solve_record(config: str):
    """A full reference solve timed on a GPU box's host (tools/ref_full_solve.py), used to check
    the bounded sample's extrapolation: the model-to-measured ratio."""
    try:
        with open(os.path.join(ROOT, "profiles", f"ref_full_solve_{config}.json")) as f:
            return json.load(f)
    except Exception:
        return None


def run_reference(args):
    """--impl reference: the reference's own CPU implementation on every host core.  C1: full
    solves, measured.  C2: bounded samples per process (H columns, capacitance rows, Cholesky,
    MINRES iterations) extrapolated with the reference's own iteration counts."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    import tempfile

    from paper_2209_02815_b200 import workload as W

    if args.config not in W.CONFIGS or args.config == "C3":
        print(json.dumps({"impl": "reference", "unavailable": f"{args.config}: the reference would hold J and H "
                          "(> 100 GB) on the host; SURVEY 8(c) reports the m=32 proxy instead"}), flush=True)
        return
    cfg = W.CONFIGS[args.config]
    inp = W.gnstep_inputs(cfg.n, cfg.m, cfg.index)
    full = 8 * cfg.m * inp.mesh.n_cells < 64e6  # C1: a whole solve takes ~0.1 s -- measure it
    iters = reference_iterations(args.config)
    alphas = list(cfg.alphas)
    if not full and any(a not in iters for a in alphas):
        raise RuntimeError(f"no reference iteration counts recorded for {args.config} (tests/golden)")
    procs, capped = ref_processes(3.2e9 if not full else 0.2e9)
    fd, path = tempfile.mkstemp(suffix=".npz", dir="/dev/shm" if os.path.isdir("/dev/shm") else None)
    os.close(fd)
    np.savez(path, J=inp.J, dm=inp.dm, dg=inp.dg)
    t_total, last = 0.0, None
    try:
        for k in range(args.warmup + args.steps):
            a = alphas[k % len(alphas)]
            v, ts, sample, kind = cpu_sample_parallel(path, cfg, a, iters.get(a), procs, 8, 8, 4, args.config, full)
            if k >= args.warmup:
                t_total += 1.0 / v  # seconds per solve of the whole host
                last = (sample, kind)
    finally:
        os.unlink(path)
    value = args.steps / t_total
    rec = full_solve_record(args.config)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (seeded {args.config} bundle)",
            "config": {"workload": f"{args.config}: unit square n={cfg.n} (N={inp.mesh.n_cells} cells, "
                                   f"K={3 * cfg.n * cfg.n + 2 * cfg.n} edges), m={cfg.m}, alpha sweep {alphas}, MINRES tol 1e-08; "
                                   f"one step = one full GN-step solve",
                       "mesh_n": cfg.n, "m": cfg.m, "alphas": alphas, "tol": 1e-8,
                       "parallelism": f"{procs} independent single-threaded reference processes"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": last[1], "sample": last[0],
                             "measured": "full solves" if full else "bounded samples, extrapolated",
                             "host": host_info(), "memory_capped": capped,
                             "iterations_source": "measured" if full else "tests/golden/c2_reference.json (reference runs)",
                             "full_solve_check": rec},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


class _Cfg:
    def __init__(self, **kw):
        self.__dict__.update(kw)


class _Inputs:
    pass


LARGE_J_BYTES = 8e9  # above this J stays on the device until the e2e arm needs a host copy


def make_problem(name, ctx, W, AmgOptions, torch):
    """Assemble the context and return (cfg, inputs, ert_info).  C1-C3: synthetic J and the
    reference's random-RHS pattern.  C4/C5: J and g from the device ERT forward model at the
    GRF log-conductivity (build time reported as t_J, outside t_norm like inversion.cpp:224),
    rhs = assemble_gn_rhs(m, 0, g, g (1 + 0.01 eps))."""
    inp = _Inputs()
    inp.J_d = None
    if name in W.ERT_CONFIGS:
        ec = W.ERT_CONFIGS[name]
        e = W.ert_inputs(name)
        inp.mesh = e.mesh
        ctx.assemble(e.mesh, AmgOptions(coarse_threshold=ec.coarse_threshold))
        ctx.set_electrodes(e.electrodes)
        ctx.use_device_pointers(True)
        model_d = torch.from_numpy(e.model).cuda()
        ctx.response_jacobian(model_d, e.survey)  # warm-up (module load, AMG)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g_d, J_d, st = ctx.response_jacobian(model_d, e.survey)
        torch.cuda.synchronize()
        t_J = time.perf_counter() - t0
        ctx.use_device_pointers(False)
        g = g_d.cpu().numpy()
        inp.J_d = J_d
        inp.J = J_d.cpu().numpy() if J_d.numel() * 8 <= LARGE_J_BYTES else None
        inp.rhs_m, inp.rhs_mref = e.model, np.zeros(e.mesh.n_cells)
        inp.rhs_g, inp.rhs_gobs = g, g * (1.0 + 0.01 * e.noise)
        m = len(g)
        cfg = _Cfg(n=ec.n, m=m, alphas=(ec.alpha,), coarse_threshold=ec.coarse_threshold, index=ec.index)
        ert = {"source": "device ERT forward model (gnw_response_jacobian)", "t_J_s": t_J,
               "electrodes": len(e.electrodes), "measurements": m, **{k: v for k, v in st.items()}}
        return cfg, inp, ert
    cfg = W.CONFIGS[name]
    K, N = W.mixed_sizes(cfg.n)
    if 8 * cfg.m * N > LARGE_J_BYTES:
        # C3: J (68.7 GB) is generated on the device; the host sees
        # it only as the e2e arm's pinned input
        inp.mesh = W.unit_square_mesh(cfg.n)
        inp.J = None
        inp.J_d = W.synthetic_jacobian_device(cfg.m, N, cfg.index, "cuda")
        torch.cuda.synchronize()
        inp.rhs_m = W.gaussian(W.seed_for(cfg.index, 2), N)
        inp.rhs_g = W.gaussian(W.seed_for(cfg.index, 3), cfg.m)
    else:
        g = W.gnstep_inputs(cfg.n, cfg.m, cfg.index)
        inp.mesh, inp.J = g.mesh, g.J
        inp.rhs_m, inp.rhs_g = g.dm, g.dg
    inp.rhs_mref, inp.rhs_gobs = np.zeros(N), np.zeros(cfg.m)
    ctx.assemble(inp.mesh, AmgOptions(coarse_threshold=cfg.coarse_threshold))
    return cfg, inp, None


def dgemm_summary(sec: float, flops: float, m: int, N: int) -> dict:
    """C = I + J H / beta: algorithmic 2 m^2 N flops, but C is symmetric and only the
    lower-triangle 128 x 128 tiles run (kernels.cu k_dgemm_nt), so the roofline fraction is the
    EXECUTED tile flops over the DMMA peak (128 flop/clk/SM x 148 SMs x 1.965 GHz)."""
    tiles = -(-m // 128)
    executed = tiles * (tiles + 1) // 2 * 128 * 128 * 2.0 * N
    return {"ms": sec * 1e3, "algorithmic_TFLOPs": flops / sec / 1e12, "executed_TFLOPs": executed / sec / 1e12,
            "frac_of_dmma_peak": executed / sec / 1e12 / 37.2, "dmma_peak_tflops": 37.2,
            "note": "frac = executed lower-triangle tile flops / DMMA peak; algorithmic = 2 m^2 N / t"}


def run_gnw(args):
    import torch

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2209_02815_b200 import AmgOptions, Context, workload as W

    tol = 1e-8
    ctx = Context(local)
    cfg, inp, ert = make_problem(args.config, ctx, W, AmgOptions, torch)
    K, N = W.mixed_sizes(cfg.n)
    alphas = list(cfg.alphas)
    info = ctx.info()

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        return max_over_ranks_dist(x, ws)

    # ---------------------------------------------------------- device-resident arm
    ctx.use_device_pointers(True)
    J_d = inp.J_d if inp.J_d is not None else torch.from_numpy(inp.J).cuda()
    dm_d = torch.from_numpy(inp.rhs_m).cuda()
    dg_d = torch.from_numpy(inp.rhs_g).cuda()
    zN = torch.from_numpy(inp.rhs_mref).cuda()
    zm = torch.from_numpy(inp.rhs_gobs).cuda()

    def solve_dev(alpha):  # the reference's GN step: inversion.cpp:244-265
        tm = ctx.set_jacobian(J_d, alpha)
        x, rep = ctx.gn_step_solve(dm_d, zN, dg_d, zm, tol=tol)
        st = ctx.stats()
        return tm, rep, st

    clk = ClockSampler(local).__enter__()  # started early: nvidia-smi start-up stays out of the timed region
    for k in range(args.warmup):
        solve_dev(alphas[k % len(alphas)])
    barrier()
    per_step = []
    launches = 0
    clk.mark()
    torch.cuda.profiler.start()  # the timed region is the profiled range (ncu --profile-from-start off)
    ctx.event_record(0)
    for k in range(args.steps):
        a = alphas[k % len(alphas)]
        tm, rep, st = solve_dev(a)
        launches += int(st["kernel_launches"]) + int(st["setup_kernel_launches"]) + 1
        per_step.append(dict(alpha=a, iterations=rep.iterations, converged=rep.converged,
                             true_rel=rep.true_relative_residual, t_H=tm["t_H"], t_C=tm["t_C"],
                             t_chol=tm["t_chol"], t_minres=st["t_minres"]))
    ctx.event_record(1)
    elapsed = ctx.event_elapsed(0, 1)
    torch.cuda.profiler.stop()
    clk.mark()
    barrier()
    value, elapsed = replica_throughput(elapsed, args.steps, ws)

    # --------------------------------------------------------------- roofline
    hbm_peak, peak_src = peaks()
    ctx.use_device_pointers(True)
    ctx.set_jacobian(J_d, 1e-2)
    b = ctx.assemble_rhs(dm_d, zN, dg_d, zm)
    ctx.minres(b, tol=tol)
    fused = ctx.stats()["fused_iterations"] > 0  # GNW_LOOP_AUTO runs tol 1e-8 on the fused/lean schedule
    lean = fused and ctx.loop_schedule() == "lean"
    kern = {}
    # launches per MINRES iteration.  Reference schedule: k_row_gemv runs twice (J zhat2, and
    # H^T v2 inside combine_prec).  The fused and lean schedules launch NO J zhat2 GEMV (u comes
    # from t' by the Woodbury identity): their one k_row_gemv is the H^T v2 pass inside
    # combine_prec, profiled alone as "row_gemv" (same kernel, same bytes) to attribute it.
    if lean:  # z2 = B (v2 - J^T t' / beta): a column sweep over J replaces the H t sweep
        per_iter = {"row_gemv": 1, "saddle_fused": 1, "combine_prec": 1, "col_sweep": 1, "finish_lean": 1,
                    "vcycle": 1, "update": 1}
    elif fused:
        per_iter = {"row_gemv": 1, "saddle_fused": 1, "combine_prec": 1, "finish_fused": 1, "vcycle": 1, "update": 1}
    else:
        per_iter = {"row_gemv": 2, "saddle": 1, "combine_prec": 1, "finish_prec": 1, "vcycle": 1, "update": 1}
    notes = {"row_gemv": ("J zhat2 and H^T v2 (the latter inside combine_prec)" if not fused else
                          "H^T v2 only -- the k_row_gemv inside combine_prec, profiled alone; no J zhat2 GEMV runs"),
             "combine_prec": "k_combine_elem + the H^T v2 k_row_gemv (not an extra sweep)",
             "vcycle": "B y' (y' = v2 - q / beta) after the column sweep" if lean else "B v2 beside H^T v2",
             "update": "standalone timing: its 0.13 GB working set is partly L2-resident; see iteration"}
    for name in per_iter:
        sec, byt = ctx.profile_kernel(name, reps=20)
        kern[name] = {"ms": sec * 1e3, "GB": byt / 1e9, "GBps": byt / sec / 1e9, "frac": byt / sec / 1e9 / hbm_peak,
                      "launches_per_iteration": per_iter[name]}
        if name in notes:
            kern[name]["note"] = notes[name]
    it_sec, it_bytes = ctx.profile_kernel("iteration")
    dg_sec, dg_flops = ctx.profile_kernel("dgemm", reps=5)
    # In-loop attribution (tools/attribute_iteration.py's method, in process): the captured loop
    # body replayed with one part left out (env GNW_EXP_SKIP, read per call); the part's marginal
    # cost beside its algorithmic bytes.  Unlike the standalone timings above, its vectors are
    # not L2-warm here (the dense sweeps evict them), so these are the honest in-loop rates.
    in_loop = {}
    try:
        skip_bits = {"vcycle": 16, "update": 128, "saddle": 2, "finish": 64, "combine": 4}
        os.environ["GNW_EXP_SKIP"] = "0"
        body_sec, _ = ctx.profile_kernel("body", reps=20)
        for part, bit in skip_bits.items():
            os.environ["GNW_EXP_SKIP"] = str(bit)
            t, _ = ctx.profile_kernel("body", reps=20)
            in_loop[part] = {"ms": (body_sec - t) * 1e3}
        byt = {"vcycle": kern["vcycle"]["GB"], "update": kern["update"]["GB"],
               "saddle": kern[sad]["GB"] if (sad := ("saddle_fused" if fused else "saddle")) in kern else None}
        for part, gb in byt.items():
            if gb and in_loop[part]["ms"] > 0:
                in_loop[part]["GB"] = gb
                in_loop[part]["GBps"] = gb / (in_loop[part]["ms"] * 1e-3)
                in_loop[part]["frac"] = in_loop[part]["GBps"] / hbm_peak
        in_loop["body_ms"] = body_sec * 1e3
    except Exception as e:  # reported, never silently replaced
        in_loop = {"failed": str(e)}
    finally:
        os.environ.pop("GNW_EXP_SKIP", None)
    # share of one iteration per kernel KIND (k_row_gemv: its own J pass + the H^T pass of combine_prec)
    sad, fin = ("saddle_fused", "finish_lean" if lean else "finish_fused") if fused else ("saddle", "finish_prec")
    kind_ms = {"row_gemv": per_iter["row_gemv"] * kern["row_gemv"]["ms"], sad: kern[sad]["ms"],
               fin: kern[fin]["ms"], "vcycle": per_iter["vcycle"] * kern["vcycle"]["ms"], "update": kern["update"]["ms"]}
    if lean:
        kind_ms["col_sweep"] = kern["col_sweep"]["ms"]
    dom = max(kind_ms, key=kind_ms.get)
    for k, v in kind_ms.items():
        kern[k]["iteration_share"] = v / (it_sec * 1e3) if it_sec else None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)
        if tj.get("config") == args.config:  # captured on that workload only
            traffic = tj["per_launch"].get(dom)
    except Exception:
        pass

    # ---------------------------------------------------------------- e2e arm
    ctx.use_device_pointers(False)
    if inp.J is None:  # large configs: J lives on the device; one pinned host copy, then free it
        J_pin = torch.empty(tuple(J_d.shape), dtype=torch.float64, pin_memory=True)
        J_pin.copy_(J_d)
        del J_d
        inp.J_d = None
        torch.cuda.empty_cache()
        J_h = J_pin.numpy()
    else:
        J_h = torch.from_numpy(inp.J).pin_memory().numpy()
    dm_h = torch.from_numpy(inp.rhs_m).pin_memory().numpy()
    dg_h = torch.from_numpy(inp.rhs_g).pin_memory().numpy()
    zN_h = torch.from_numpy(inp.rhs_mref).pin_memory().numpy()
    zm_h = torch.from_numpy(inp.rhs_gobs).pin_memory().numpy()

    x_h = torch.empty(K + N, dtype=torch.float64, pin_memory=True).numpy()   # solution (D2H)

    def solve_host(alpha, prefetch_next):
        # the reference's GN step (inversion.cpp:244-265): build_woodbury_preconditioner, then
        # b = assemble_gn_rhs(...), x0 = 0, minres -- the last three as one C-ABI call
        # (gnw_gn_step_solve): host m, m_ref, g, g_obs in, host x out
        ctx.set_jacobian(J_h, alpha)  # takes the staged copy when the previous step prefetched it
        if prefetch_next:  # the next step's J crosses PCIe during this step's MINRES
            ctx.prefetch_jacobian(J_h)
        x, rep = ctx.gn_step_solve(dm_h, zN_h, dg_h, zm_h, tol=tol, out=x_h)
        return x, rep

    solve_host(alphas[0], False)  # nothing staged when the timed region opens: step 0 copies J itself
    barrier()
    ctx.event_record(2)
    e2e_iters = []
    for k in range(args.steps):
        x_h, rep_h = solve_host(alphas[k % len(alphas)], k + 1 < args.steps)
        e2e_iters.append(rep_h.iterations)  # host-side scalars only: no device work added
    ctx.event_record(3)
    e2e_elapsed = max_over_ranks(ctx.event_elapsed(2, 3))
    barrier()
    h2d = 8 * (cfg.m * N + 2 * N + 2 * cfg.m)               # J, m, m_ref, g, g_obs
    d2h = 8 * (K + N) + 8 * 2 * (rep_h.iterations + 1)      # x, residual histories

    # ---------------------------------------------------------- CPU baseline
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and 8 * cfg.m * N > LARGE_J_BYTES:
        cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
               "sample": f"not run: the reference holds J and H on the host ({16 * cfg.m * N / 1e9:.0f} GB), "
                         f"beside the e2e arm's pinned J (SURVEY.md 8(c): C3/C5 full m infeasible on the host)"}
    elif rank == 0 and ws == 1 and not args.no_cpu_baseline:
        a_cpu = 1e-2 if 1e-2 in alphas else alphas[0]
        # the reference's own iteration count where a reference run is recorded, else the GPU's
        # (iterations match within +-1: tests/test_gpu_golden.py)
        it_use = reference_iterations(args.config).get(a_cpu) or next(
            s["iterations"] for s in per_step if s["alpha"] == a_cpu)
        try:
            v, t_est, s, sample, kind = cpu_sample(cfg, inp, a_cpu, it_use, label=args.config)
            cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": kind, "sample": sample, "host": host_info()}
        except Exception as e:  # reported, never silently replaced
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": f"synthetic (seeded {args.config} bundle)",
            "config": {"workload": f"{args.config}: unit square n={cfg.n} (N={N} cells, K={K} edges), m={cfg.m}, "
                                   f"alpha sweep {alphas}, MINRES tol {tol}; one step = one full GN-step solve",
                       "mesh_n": cfg.n, "m": cfg.m, "alphas": alphas, "tol": tol,
                       "parallelism": f"replicas x{ws}",
                       "l2": f"no flush: per-solve inputs (J {8 * cfg.m * N / 1e9:.2f} GB + H {8 * cfg.m * N / 1e9:.2f} GB) exceed the 126 MB L2",
                       "amg_levels": info["n_levels"], "coarse_n": info["coarse_n"],
                       "jacobian": ert if ert else "synthetic U diag(10^(-4k/m)) V^T (workload.py)"},
            "roofline": {"bound": "hbm", "kernel": KERNEL_NAMES.get(dom, "k_" + dom),
                         "loop_schedule": ctx.loop_schedule() + (" (GNW_LOOP_AUTO at tol >= 1e-8)" if fused else ""), "achieved": kern[dom]["GBps"], "peak": hbm_peak,
                         "unit": "GB/s", "frac": kern[dom]["frac"], "traffic": traffic,
                         "peak_source": peak_src,
                         "peak_note": "hbm_gbs is a COPY bandwidth (read + write); the dominant kernels are read-only "
                                      "streams, which reach up to ~7.1 TB/s on this part, so frac can exceed 1",
                         "algorithmic_bytes_per_launch": kern[dom]["GB"] * 1e9,
                         "iteration_share": kern[dom]["iteration_share"],
                         "dmma_peak_tflops": 37.2,
                         "iteration": {"ms": it_sec * 1e3, "GB": it_bytes / 1e9,
                                       "GBps": it_bytes / it_sec / 1e9 if it_sec else None,
                                       "frac": it_bytes / it_sec / 1e9 / hbm_peak if it_sec else None},
                         "kernels": kern,
                         "in_loop": in_loop,
                         "dgemm": dgemm_summary(dg_sec, dg_flops, cfg.m, N)},
            "cpu_baseline": cpu,
            "e2e": {"value": ws * args.steps / e2e_elapsed, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "iterations": e2e_iters,
                    "loop_restarts": ctx.stats()["loop_restarts"]},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "phases": per_step,
        }
    clk.__exit__(None, None, None)
    ctx.close()
    J_d = inp = None  # free the replica's device inputs before the partitioned leg
    torch.cuda.empty_cache()
    # The north star's strong-scaling case: ONE C3 solve row-partitioned over the N GPUs (SURVEY
    # 8(e)).  Reported beside the replica metric when N > 1 (or GNW_BENCH_PARTITIONED=1), so the
    # driver's 1/2/4/8-GPU runs also trace the partitioned curve.
    part_cfg = os.environ.get("GNW_BENCH_PARTITIONED_CONFIG", "C3")
    if ws > 1 or os.environ.get("GNW_BENCH_PARTITIONED") == "1":
        # watchdog: a rank that fails inside a collective leaves the others waiting; the replica
        # line must still be printed, so on timeout rank 0 prints it (partitioned: failed) and
        # every rank leaves without the NCCL teardown
        limit = float(os.environ.get("GNW_BENCH_PARTITIONED_TIMEOUT", "600"))

        def give_up():
            if rank == 0:
                line["partitioned"] = {"failed": f"timeout after {limit:.0f} s"}
                print(json.dumps(line), flush=True)
            os._exit(0)

        dog = threading.Timer(limit, give_up)
        dog.daemon = True
        dog.start()
        try:
            part = partitioned_leg(part_cfg, steps=2, warmup=1)
        except Exception as e:  # reported, never silently replaced
            part = {"failed": f"{type(e).__name__}: {e}"}
            if ws > 1:  # the other ranks may be inside a collective: no barrier, no teardown
                dog.cancel()
                if rank == 0:
                    line["partitioned"] = part
                    print(json.dumps(line), flush=True)
                os._exit(0)
        dog.cancel()
        if rank == 0:
            line["partitioned"] = part
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def partitioned_leg(config: str, steps: int, warmup: int, tol: float = 1e-8) -> dict:
    """ONE GN-step solve of `config` row-partitioned over the torch.distributed world (one rank
    per GPU, NCCL inside libgnw): each rank generates its J column slice on its device
    (distributed CholeskyQR2), the MINRES vectors / SpMV / fine V-cycle levels run on its mesh
    rows with halo exchanges.  Collective; returns the summary (max-over-ranks device times)."""
    import torch

    from paper_2209_02815_b200 import (AmgOptions, Context, nccl_unique_id, partitioned_from_torch_distributed,
                                       workload as W)

    ws, rank, local = dist_env()
    cfg = W.CONFIGS[config]
    K, N = W.mixed_sizes(cfg.n)
    t_setup0 = time.perf_counter()
    ctx = partitioned_from_torch_distributed(local) if ws > 1 else Context.partitioned(0, 1, nccl_unique_id(), local)
    ctx.assemble(W.unit_square_mesh(cfg.n), AmgOptions(coarse_threshold=cfg.coarse_threshold))
    part = ctx.partition()
    allreduce = (lambda t: torch.distributed.all_reduce(t)) if ws > 1 else None
    J_d = W.synthetic_jacobian_slice(cfg.m, N, cfg.index, part["c_lo"], part["c_hi"], "cuda", allreduce=allreduce)
    t_setup = time.perf_counter() - t_setup0
    ctx.use_device_pointers(True)
    dm_d = torch.from_numpy(W.gaussian(W.seed_for(cfg.index, 2), N)).cuda()
    dg_d = torch.from_numpy(W.gaussian(W.seed_for(cfg.index, 3), cfg.m)).cuda()
    zN = torch.zeros(N, dtype=torch.float64, device="cuda")
    zm = torch.zeros(cfg.m, dtype=torch.float64, device="cuda")
    alphas = list(cfg.alphas)

    def solve(alpha):
        tm = ctx.set_jacobian(J_d, alpha)
        b = ctx.assemble_rhs(dm_d, zN, dg_d, zm)
        x, rep = ctx.minres(b, tol=tol)
        return tm, rep, ctx.stats()

    for k in range(warmup):
        solve(alphas[k % len(alphas)])
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    ctx.event_record(0)
    phases = []
    for k in range(steps):
        a = alphas[k % len(alphas)]
        tm, rep, st = solve(a)
        phases.append(dict(alpha=a, iterations=rep.iterations, converged=rep.converged,
                           true_rel=rep.true_relative_residual, t_minres=st["t_minres"],
                           ms_per_iteration=1e3 * st["t_minres"] / max(rep.iterations, 1),
                           exchanges=st["comm_calls"], exchange_MB=st["comm_bytes"] / 1e6, **tm))
    ctx.event_record(1)
    elapsed = max_over_ranks_dist(ctx.event_elapsed(0, 1), ws)
    it_ms = max_over_ranks_dist(phases[-1]["ms_per_iteration"], ws)
    info = dict(own_cells=part["c_hi"] - part["c_lo"])
    ctx.close()
    del J_d
    torch.cuda.empty_cache()
    # per-rank roofline of the lean iteration: (B_iter - 16 m N + B_V) / P bytes per rank
    hbm_peak, _ = peaks()
    bytes_rank = 8.0 * 2 * cfg.m * N / ws + 8 * 40 * (K + N) / ws  # the two dense sweeps + vector traffic
    return {"metric": METRIC, "value": steps / elapsed, "unit": UNIT, "n_gpus": ws, "scaling": "strong",
            "workload": f"{config}: unit square n={cfg.n} (N={N}, K={K}), m={cfg.m}, alpha {alphas}, tol {tol}; "
                        f"one GN-step solve row-partitioned over {ws} GPU(s)",
            "ms_per_solve": 1e3 * elapsed / steps, "ms_per_iteration": it_ms, "setup_s_rank0": t_setup,
            "rank0": info, "phases": phases,
            "per_rank_roofline": {"bytes_per_iteration_GB": bytes_rank / 1e9,
                                  "GBps": bytes_rank / (it_ms * 1e-3) / 1e9,
                                  "frac": bytes_rank / (it_ms * 1e-3) / 1e9 / hbm_peak,
                                  "note": "dense sweeps (16 m N / P) + ~40 (K + N) / P vector bytes; V-cycle excluded"}}


def run_partitioned(args):
    """--partitioned: ONE GN-step solve split over the N GPUs by mesh rows (SURVEY 8(e), C3/C5
    scale; `scaling` strong)."""
    import torch

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    clk = ClockSampler(local).__enter__()
    clk.mark()
    res = partitioned_leg(args.config, args.steps, args.warmup)
    clk.mark()
    clk.__exit__(None, None, None)
    if rank == 0:
        line = {"metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": res["ms_per_solve"], "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": f"synthetic (seeded {args.config} bundle, J slices generated per rank on the device)",
                "config": {"workload": res["workload"], "parallelism": f"row-partitioned x{ws} (NCCL)"},
                "partitioned": res, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="gnw", choices=["gnw", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--partitioned", action="store_true",
                    help="split ONE solve over the N GPUs by cell columns (C3-scale; NCCL inside libgnw)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.partitioned:
        run_partitioned(args)
    else:
        run_gnw(args)


if __name__ == "__main__":
    main()
