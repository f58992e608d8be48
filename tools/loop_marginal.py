"""Marginal cost of one MINRES iteration inside the conditional-graph loop: (t(tol_a) - t(tol_b))
/ (it_a - it_b), which removes the per-solve fixed work (initial residual, first preconditioner
apply, verification) from the per-iteration figure.

    python tools/loop_marginal.py C1 C2
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
from paper_2209_02815_b200 import AmgOptions, Context, workload as W  # noqa: E402

for name in sys.argv[1:] or ["C2"]:
    cfg = W.CONFIGS[name]
    inp = W.gnstep_inputs(cfg.n, cfg.m, cfg.index)
    ctx = Context(0)
    ctx.assemble(inp.mesh, AmgOptions(coarse_threshold=cfg.coarse_threshold))
    ctx.set_jacobian(inp.J, cfg.alphas[0])
    b = ctx.assemble_rhs(inp.dm, np.zeros(ctx.N), inp.dg, np.zeros(cfg.m))
    ctx.minres(b, tol=1e-8)
    res = {}
    for tol in (1e-4, 1e-8):
        ts = []
        for _ in range(3):
            _, rep = ctx.minres(b, tol=tol)
            ts.append(ctx.stats()["t_minres"])
        res[tol] = (rep.iterations, min(ts))
    (ia, ta), (ib, tb) = res[1e-8], res[1e-4]
    body, _ = ctx.profile_kernel("body", reps=50)
    print(f"{name}: {ia} it {1e3 * ta:.3f} ms, {ib} it {1e3 * tb:.3f} ms -> marginal {1e3 * (ta - tb) / (ia - ib):.4f} "
          f"ms/it; replayed body {1e3 * body:.4f} ms; fixed per solve {1e3 * (ta - ia * (ta - tb) / (ia - ib)):.3f} ms")
