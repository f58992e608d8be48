"""Per-iteration hot kernels of the C2 MINRES loop launched standalone (gnw_profile_kernel),
bracketed by cudaProfilerStart/Stop for ncu --profile-from-start off.  The loop itself runs
inside a conditional CUDA graph, whose kernels ncu does not list individually.

    python tools/profile_kernels.py [--config C2] [--reps 3]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_02815_b200 import AmgOptions, Context, workload as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--kernels", default="row_gemv,saddle,combine_prec,finish_prec,vcycle,update")
args = ap.parse_args()

cfg = W.CONFIGS[args.config]
inp = W.gnstep_inputs(cfg.n, cfg.m, cfg.index)
ctx = Context(0)
ctx.assemble(inp.mesh, AmgOptions(coarse_threshold=cfg.coarse_threshold))
ctx.use_device_pointers(True)
J = torch.from_numpy(inp.J).cuda()
ctx.set_jacobian(J, 1e-2)
names = args.kernels.split(",")
for nm in names:  # warm-up (module load) outside the profiled range
    ctx.profile_kernel(nm, reps=1)
torch.cuda.synchronize()
torch.cuda.profiler.start()
res = {nm: ctx.profile_kernel(nm, reps=args.reps) for nm in names}
torch.cuda.synchronize()
torch.cuda.profiler.stop()
for nm, (sec, alg) in res.items():
    print(f"{nm:14s} {1e3 * sec:8.3f} ms  {alg / 1e9:7.3f} GB  {alg / sec / 1e9:8.1f} GB/s")
