"""MINRES loop schedules side by side on a config (gnw.h GNW_LOOP_*): iterations, restarts,
true residuals, timings, and each schedule's distance from the reference schedule's solution
(tol 1e-8 and 1e-12).

    python tools/check_fused.py [--config C2] [--modes reference,fused,lean] [--n N --m M]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2209_02815_b200 import AmgOptions, Context, workload as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--modes", default="reference,fused,lean")
ap.add_argument("--tols", default="1e-8,1e-12")
args = ap.parse_args()
cfg = W.CONFIGS[args.config]
inp = W.gnstep_inputs(cfg.n, cfg.m, cfg.index)
ref = {}
try:
    rec = json.load(open(os.path.join(ROOT, "tests", "golden", "c2_reference.json")))
    ref = {r["alpha"]: r["iterations"] for r in rec["runs"]} if args.config == "C2" else {}
except Exception:
    pass
ctx = Context(0)
ctx.assemble(inp.mesh, AmgOptions(coarse_threshold=cfg.coarse_threshold))
ctx.use_device_pointers(True)
J = torch.from_numpy(inp.J).cuda()
dm = torch.from_numpy(inp.dm).cuda()
dg = torch.from_numpy(inp.dg).cuda()
zN = torch.zeros(inp.mesh.n_cells, dtype=torch.float64, device="cuda")
zm = torch.zeros(cfg.m, dtype=torch.float64, device="cuda")
modes = args.modes.split(",")
tols = [float(t) for t in args.tols.split(",")]
for a in cfg.alphas:
    out = {}
    for mode in modes:
        ctx.set_loop_mode(mode)
        ctx.set_jacobian(J, a)
        b = ctx.assemble_rhs(dm, zN, dg, zm)
        for tol in tols:
            ctx.minres(b, tol=tol)  # warm
            torch.cuda.synchronize()
            r0 = ctx.stats()["loop_restarts"]
            t0 = time.perf_counter()
            x, rep = ctx.minres(b, tol=tol)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            out[(mode, tol)] = (x.cpu().numpy(), rep, dt, ctx.stats()["loop_restarts"] - r0)
    for tol in tols:
        xr = out[(modes[0], tol)][0]
        parts = []
        for mode in modes:
            x, rep, dt, rs = out[(mode, tol)]
            d = np.linalg.norm(x - xr) / np.linalg.norm(xr)
            parts.append(f"{mode} {rep.iterations} it ({rs} rs) {1e3 * dt:.1f} ms "
                         f"{1e3 * dt / max(rep.iterations, 1):.3f} ms/it true {rep.true_relative_residual:.2e} d {d:.1e}")
        print(f"alpha={a:g} tol={tol:g}: " + " | ".join(parts)
              + (f" | reference run {ref[a]}" if tol == 1e-8 and a in ref else ""), flush=True)
