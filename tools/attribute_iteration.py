"""Attribute the MINRES iteration time to its parts: the loop body is captured once and
replayed (gnw_profile_kernel GNW_K_BODY) with parts left out via GNW_EXP_SKIP.  The numbers
are timings of a numerically meaningless body -- attribution only, never a result.

    python tools/attribute_iteration.py [--config C2]
"""
import argparse
import os
import subprocess
import sys

PARTS = {"J row GEMV": 1, "saddle (J^T u)": 2, "combine elem": 4, "H^T y GEMV": 8, "V-cycle": 16,
         "C^-1 apply": 32, "finish (H t)": 64, "update": 128, "col sweep (lean)": 256}

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, os.getcwd())
    import numpy as np
    from paper_2209_02815_b200 import AmgOptions, Context, workload as W
    cfg = W.CONFIGS[sys.argv[2]]
    inp = W.gnstep_inputs(cfg.n, cfg.m, cfg.index)
    ctx = Context(0)
    ctx.assemble(inp.mesh, AmgOptions(coarse_threshold=cfg.coarse_threshold))
    ctx.set_jacobian(inp.J, cfg.alphas[0])
    b = ctx.assemble_rhs(inp.dm, np.zeros(ctx.N), inp.dg, np.zeros(cfg.m))
    ctx.minres(b, tol=1e-8)
    sec, _ = ctx.profile_kernel("body", reps=50)
    it, _ = ctx.profile_kernel("iteration")
    print(f"{1e3 * sec:.4f} {1e3 * it:.4f}")
    sys.exit(0)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
args = ap.parse_args()


def run(mask):
    env = dict(os.environ, GNW_EXP_SKIP=str(mask))
    out = subprocess.run([sys.executable, __file__, "--child", args.config], env=env, capture_output=True,
                         text=True, check=True).stdout.split()
    return float(out[0]), float(out[1])


full, it = run(0)
print(f"{args.config}: loop iteration {it:.4f} ms; replayed body {full:.4f} ms")
for name, bit in PARTS.items():
    t, _ = run(bit)
    print(f"  without {name:16s} {t:.4f} ms  (part costs {full - t:+.4f} ms)")
print(f"  everything skipped {run(511)[0]:.4f} ms (graph launch floor)")
