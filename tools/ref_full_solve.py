"""Times ONE full reference GN-step solve (oracle/_ref, the unmodified reference) on this host
next to the bounded sample bench.py's CPU legs extrapolate from, and writes the
model-to-measured ratio to profiles/ref_full_solve_<config>.json (read back by
bench.py --impl reference as cpu_baseline.full_solve_check).  Run it on the GPU box's host:

    python tools/ref_full_solve.py [--config C2] [--alpha 1e-2]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import bench  # noqa: E402
import orc  # noqa: E402
from paper_2209_02815_b200 import workload as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--alpha", type=float, default=1e-2)
    args = ap.parse_args()
    cfg = W.CONFIGS[args.config]
    inp = W.gnstep_inputs(cfg.n, cfg.m, cfg.index)
    iters = bench.reference_iterations(args.config).get(args.alpha)
    # the bounded sample exactly as bench.py's legs run it (single process, idle host)
    t0 = time.time()
    v, t_est, parts, sample, kind = bench.cpu_sample(cfg, inp, args.alpha, iters, k_cols=8, k_rows=8, k_iters=4,
                                                      label=args.config)
    t_sample = time.time() - t0
    # the full solve: set_jacobian + assemble_gn_rhs + minres (inversion.cpp:242-271)
    o = orc.Oracle("reference")
    p = orc.Problem.mixed(o, inp.mesh, orc.AmgOpts.make(coarse_threshold=cfg.coarse_threshold))
    t0 = time.time()
    tim = p.set_jacobian(inp.J, args.alpha)
    b = p.assemble_rhs(inp.dm, np.zeros(p.N), inp.dg, np.zeros(cfg.m))
    t1 = time.time()
    x, rep = p.minres(b, tol=1e-8)
    t_norm = time.time() - t0
    out = dict(config=args.config, alpha=args.alpha, host=bench.host_info(), kind=kind,
               measured_t_norm_s=t_norm, measured_iterations=rep["iterations"], measured_t_minres_s=time.time() - t1,
               measured_timings=tim, sample_t_norm_s=t_est, sample_parts=parts, sample_wall_s=t_sample,
               sample_iterations=iters, model_to_measured=t_est / t_norm,
               when=time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()))
    path = os.path.join(ROOT, "profiles", f"ref_full_solve_{args.config}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"ref_full_solve_{args.config}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
