#!/bin/bash
# Kernel timings vs. row padding of the owned J / Ht copies (host-pointer J).
for p in 0 16 64 256; do
  echo "pad=$p"
  GNW_PAD=$p python - <<'PY'
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2209_02815_b200 import AmgOptions, Context, workload as W
cfg = W.CONFIGS["C2"]; inp = W.gnstep_inputs(cfg.n, cfg.m, cfg.index)
ctx = Context(0); ctx.assemble(inp.mesh, AmgOptions())
ctx.set_jacobian(inp.J, 1e-2)
for nm in ("row_gemv", "saddle", "combine_prec", "finish_prec"):
    ctx.profile_kernel(nm, reps=2); s, a = ctx.profile_kernel(nm, reps=20)
    print(f"  {nm:14s} {1e3*s:7.3f} ms {a/s/1e9:7.1f} GB/s")
ctx.set_loop_mode(True); ctx.set_jacobian(inp.J, 1e-2)
b = ctx.assemble_rhs(inp.dm, np.zeros(ctx.N), inp.dg, np.zeros(cfg.m))
for fused in (False, True):
    ctx.set_loop_mode(fused); ctx.set_jacobian(inp.J, 1e-2); ctx.minres(b, tol=1e-8)
    x, rep = ctx.minres(b, tol=1e-8); st = ctx.stats()
    print(f"  fused={fused} minres {1e3*st['t_minres']:.1f} ms {rep.iterations} it -> {1e3*st['t_minres']/rep.iterations:.3f} ms/it")
PY
done
