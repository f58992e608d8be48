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
ap.add_argument("--n", type=int, default=0, help="override: mesh n (J generated on the device)")
ap.add_argument("--m", type=int, default=0, help="override: rows of J")
ap.add_argument("--coarse-threshold", type=int, default=64)
args = ap.parse_args()

ctx = Context(0)
if args.n:  # e.g. C5 shapes: --n 1024 --m 3780 --coarse-threshold 1024
    mesh = W.unit_square_mesh(args.n)
    ctx.assemble(mesh, AmgOptions(coarse_threshold=args.coarse_threshold))
    J = W.synthetic_jacobian_device(args.m, mesh.n_cells, 9, "cuda")
else:
    cfg = W.CONFIGS[args.config]
    inp = W.gnstep_inputs(cfg.n, cfg.m, cfg.index)
    ctx.assemble(inp.mesh, AmgOptions(coarse_threshold=cfg.coarse_threshold))
    J = torch.from_numpy(inp.J).cuda()
ctx.use_device_pointers(True)
ctx.set_jacobian(J, 1e-2)
if args.n == 0:  # one solve first: "iteration" is the last solve's time per MINRES iteration
    b = ctx.assemble_rhs(torch.from_numpy(inp.dm).cuda(), torch.zeros(inp.mesh.n_cells, dtype=torch.float64, device="cuda"),
                         torch.from_numpy(inp.dg).cuda(), torch.zeros(cfg.m, dtype=torch.float64, device="cuda"))
    for _ in range(2):
        x, rep = ctx.minres(b, tol=1e-8)
    print(f"solve: {rep.iterations} iterations, schedule {ctx.loop_schedule()}, info {ctx.info()}")
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
