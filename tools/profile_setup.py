"""One Woodbury setup (set_jacobian: H, C, chol C, C^-1) bracketed by cudaProfilerStart/Stop,
for an ncu launch list of the setup kernels.

    python tools/profile_setup.py --n 256 --m 868
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_02815_b200 import AmgOptions, Context, workload as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--m", type=int, default=868)
ap.add_argument("--coarse-threshold", type=int, default=64)
args = ap.parse_args()
mesh = W.unit_square_mesh(args.n)
ctx = Context(0)
ctx.assemble(mesh, AmgOptions(coarse_threshold=args.coarse_threshold))
J = W.synthetic_jacobian_device(args.m, mesh.n_cells, 9, "cuda")
ctx.use_device_pointers(True)
ctx.set_jacobian(J, 1e-2)
torch.cuda.synchronize()
torch.cuda.profiler.start()
t = ctx.set_jacobian(J, 1e-2)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print({k: round(v * 1e3, 3) for k, v in t.items()}, "ms")
