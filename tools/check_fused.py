"""Reference-schedule vs fused MINRES loop on a config: iterations, residuals, timings,
and the distance between the two solutions (tol 1e-8 and 1e-12).

    python tools/check_fused.py [--config C2]
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
for a in cfg.alphas:
    out = {}
    for fused in (False, True):
        ctx.set_loop_mode(fused)
        ctx.set_jacobian(J, a)
        b = ctx.assemble_rhs(dm, zN, dg, zm)
        for tol in (1e-8, 1e-12):
            ctx.minres(b, tol=tol)  # warm
            torch.cuda.synchronize()
            r0 = ctx.stats()["loop_restarts"]
            t0 = time.perf_counter()
            x, rep = ctx.minres(b, tol=tol)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            rep.restarts = ctx.stats()["loop_restarts"] - r0
            out[(fused, tol)] = (x.cpu().numpy(), rep, dt)
    for tol in (1e-8, 1e-12):
        xr, rr, tr = out[(False, tol)]
        xf, rf, tf = out[(True, tol)]
        d = np.linalg.norm(xr - xf) / np.linalg.norm(xr)
        print(f"alpha={a:g} tol={tol:g}: ref-loop {rr.iterations} it {1e3 * tr:.1f} ms true {rr.true_relative_residual:.2e} | "
              f"fused {rf.iterations} it ({rf.restarts} restarts) {1e3 * tf:.1f} ms true {rf.true_relative_residual:.2e} | rel diff {d:.2e}"
              + (f" | reference {ref[a]}" if tol == 1e-8 and a in ref else ""), flush=True)
