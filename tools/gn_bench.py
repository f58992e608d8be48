"""Woodbury- vs Laplace-preconditioned Gauss-Newton on the device, written in the reference
`bench` command's CSV layout (proj/tools/main.cpp:252-310):
    nele,N,M,algo,step,n_iter,t_H,t_C,t_chol,t_norm,status

The reference's bench uses its half-disk mesher, pole-dipole survey and checkerboard model
(out of scope here); this driver uses the BASELINE-style unit-square
meshes, the adjacent-pair dipole-dipole survey and the seeded GRF model (workload.py), with
noise-free synthetic data from the device forward model at the true model, like the reference.

    python tools/gn_bench.py [--out profiles/r01_gn_bench.csv] [--steps 2] [--beta 0.1]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_02815_b200 import Context, workload as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="profiles/r01_gn_bench.csv")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--beta", type=float, default=0.1)
ap.add_argument("--tol", type=float, default=1e-7)
ap.add_argument("--cases", default="64:8,128:16,256:32")
args = ap.parse_args()

rows = ["nele,N,M,algo,step,n_iter,t_H,t_C,t_chol,t_norm,status"]
for case in args.cases.split(","):
    n, nele = (int(v) for v in case.split(":"))
    mesh = W.unit_square_mesh(n)
    step = max(1, (n - 8) // nele)
    nodes = np.array([4 + step * e for e in range(nele)], dtype=np.int64)
    sv = W.ert_survey(nele, mesh.vertices[nodes, 0])
    truth = W.conductivity_model(mesh, 3)
    ctx = Context(0)
    ctx.assemble(mesh)
    ctx.set_electrodes(nodes)
    g_obs, _, _ = ctx.response_jacobian(truth, sv)
    m0 = np.full(mesh.n_cells, float(np.mean(truth)))
    for algo in ("woodbury", "laplace"):
        try:
            _, rep = ctx.gauss_newton(m0, m0, sv, g_obs, beta=args.beta, max_outer_steps=args.steps,
                                      minres_tol=args.tol, algorithm=algo)
            for k, s in enumerate(rep["steps"]):
                rows.append(f"{nele},{mesh.n_cells},{len(g_obs)},{algo},{k + 1},{s['minres_iters']},"
                            f"{s['t_H']:.6g},{s['t_C']:.6g},{s['t_chol']:.6g},{s['t_norm']:.6g},ok")
            print(f"bench nele={nele} algo={algo} done: misfit {rep['steps'][0]['misfit']:.4g} -> "
                  f"{rep['final_misfit']:.4g}", flush=True)
        except Exception as e:  # noqa: BLE001 -- recorded like the reference's bench
            rows.append(f"{nele},0,0,{algo},0,0,0,0,0,0,error")
            print(f"bench nele={nele} algo={algo} failed: {e}", file=sys.stderr)
    ctx.close()
with open(args.out, "w") as f:
    f.write("\n".join(rows) + "\n")
print("bench ->", args.out)
print("\n".join(rows))
