"""MINRES iteration counts and residual-history tails of one proxy problem on every loop schedule
and coarse mode (diagnostics for tests/test_gpu_baseline_parity.py).

    python tools/diag_iters.py [--n 1024] [--thr 1024] [--index 4] [--alpha 1e-3] [--m 32]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2209_02815_b200 import AmgOptions, Context, workload as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--thr", type=int, default=1024)
ap.add_argument("--index", type=int, default=4)
ap.add_argument("--alpha", type=float, default=1e-3)
ap.add_argument("--m", type=int, default=32)
ap.add_argument("--tol", type=float, default=1e-8)
args = ap.parse_args()

inp = W.gnstep_inputs(args.n, args.m, args.index)
out = {}
for exact in (False, True):
    c = Context(0)
    c.set_coarse_mode(exact)
    c.assemble(inp.mesh, AmgOptions(coarse_threshold=args.thr))
    c.set_jacobian(inp.J, args.alpha)
    b = c.assemble_rhs(inp.dm, np.zeros(c.N), inp.dg, np.zeros(args.m))
    for mode in ("reference", "fused", "lean"):
        c.set_loop_mode(mode)
        x, rep = c.minres(b, tol=args.tol)
        key = f"{'exact' if exact else 'default'}/{mode}"
        out[key] = dict(iterations=rep.iterations, true_rel=rep.true_relative_residual,
                        restarts=c.stats()["loop_restarts"], hist_e=rep.relative_residuals.tolist(),
                        hist_p=rep.pnorm_relative_residuals.tolist())
        h = rep.relative_residuals
        print(key, rep.iterations, f"true {rep.true_relative_residual:.3e}", "tail", np.array2string(h[-6:], precision=3),
              flush=True)
    c.close()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", f"diag_iters_n{args.n}.json"), "w") as f:
    json.dump(out, f)
