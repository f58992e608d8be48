"""Full reference GN-step solves on BASELINE config C2 (512x512 unit square, m = 256, alpha sweep).

Runs the UNMODIFIED reference (oracle/_ref/libertinv_ref.so, built from /root/reference
by oracle/Makefile) through build_woodbury_preconditioner + assemble_gn_rhs + minres on the
seeded C2 bundle (paper_2209_02815_b200.workload), one process per alpha, and writes
tests/golden/c2_reference.json: per alpha the MINRES iteration count, the true relative
residual and the reference's own timers (t_H, t_C, t_chol, t_minres, t_norm).

bench.py's CPU legs extrapolate their bounded samples with these iteration counts, and
tests check that the GPU path reproduces them within +-1.  Takes ~3 minutes per alpha.
"""
import json
import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def run(alpha):
    import numpy as np
    import orc
    from paper_2209_02815_b200 import workload as W

    cfg = W.CONFIGS["C2"]
    inp = W.gnstep_inputs(cfg.n, cfg.m, cfg.index)
    o = orc.Oracle("reference")
    t0 = time.time()
    p = orc.Problem.mixed(o, inp.mesh, orc.AmgOpts.make(coarse_threshold=cfg.coarse_threshold))
    t_setup = time.time() - t0
    t0 = time.time()
    tim = p.set_jacobian(inp.J, alpha)
    b = p.assemble_rhs(inp.dm, np.zeros(p.N), inp.dg, np.zeros(cfg.m))
    t1 = time.time()
    x, rep = p.minres(b, tol=1e-8)
    t_minres = time.time() - t1
    t_norm = time.time() - t0
    return dict(alpha=alpha, iterations=rep["iterations"], converged=rep["converged"],
                true_relative_residual=rep["true_relative_residual"], t_setup_once=t_setup,
                t_H=tim["t_H"], t_C=tim["t_C"], t_chol=tim["t_chol"], t_minres=t_minres, t_norm=t_norm,
                x_norm=float(np.linalg.norm(x)), x_head=[float(v) for v in x[:4]])


if __name__ == "__main__":
    alphas = [1e-4, 1e-3, 1e-2, 1e-1, 1.0]
    with mp.get_context("spawn").Pool(len(alphas)) as pool:
        res = pool.map(run, alphas)
    out = dict(config="C2", n=512, m=256, tol=1e-8, host=os.uname().nodename, cores_per_run=1,
               note="reference library single-threaded; 5 alphas run concurrently on one host",
               runs=res)
    with open(os.path.join(HERE, "c2_reference.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))
