"""One C2 GN-step solve bracketed by cudaProfilerStart/Stop, for ncu --profile-from-start off.

    python tools/profile_one.py [--config C2] [--alpha 1e-2]

A warm-up solve runs first (outside the profiled range) so module loading, graph
instantiation and buffer allocation are excluded.
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_02815_b200 import AmgOptions, Context, workload as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--alpha", type=float, default=1e-2)
ap.add_argument("--tol", type=float, default=1e-8)
args = ap.parse_args()

cfg = W.CONFIGS[args.config]
inp = W.gnstep_inputs(cfg.n, cfg.m, cfg.index)
ctx = Context(0)
ctx.assemble(inp.mesh, AmgOptions(coarse_threshold=cfg.coarse_threshold))
ctx.use_device_pointers(True)
J = torch.from_numpy(inp.J).cuda()
dm = torch.from_numpy(inp.dm).cuda()
dg = torch.from_numpy(inp.dg).cuda()
zN = torch.zeros(inp.mesh.n_cells, dtype=torch.float64, device="cuda")
zm = torch.zeros(cfg.m, dtype=torch.float64, device="cuda")


def solve():
    t = ctx.set_jacobian(J, args.alpha)
    b = ctx.assemble_rhs(dm, zN, dg, zm)
    x, rep = ctx.minres(b, tol=args.tol)
    return t, rep


solve()
torch.cuda.synchronize()
torch.cuda.profiler.start()
t0 = time.perf_counter()
t, rep = solve()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
torch.cuda.profiler.stop()
st = ctx.stats()
print(f"{args.config} alpha={args.alpha}: {rep.iterations} iterations, wall {1e3 * wall:.1f} ms, "
      f"t_H {1e3 * t['t_H']:.2f} t_C {1e3 * t['t_C']:.2f} t_chol {1e3 * t['t_chol']:.2f} "
      f"t_minres {1e3 * st['t_minres']:.2f} ms, launches {st['kernel_launches']}+{st['setup_kernel_launches']}")
