"""C1 solve time under the V-cycle tail / fused-loop variants (env GNW_TAIL_CLUSTER)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2209_02815_b200 import AmgOptions, Context, workload as W
for name in sys.argv[1:] or ["C1"]:
    cfg = W.CONFIGS[name]; inp = W.gnstep_inputs(cfg.n, cfg.m, cfg.index)
    ctx = Context(0); ctx.assemble(inp.mesh, AmgOptions(coarse_threshold=cfg.coarse_threshold))
    for fused in (False, True):
        ctx.set_loop_mode(fused)
        ctx.set_jacobian(inp.J, cfg.alphas[0])
        b = ctx.assemble_rhs(inp.dm, np.zeros(ctx.N), inp.dg, np.zeros(cfg.m))
        ctx.minres(b, tol=1e-8)
        x, rep = ctx.minres(b, tol=1e-8); st = ctx.stats()
        print(f"{name} tail={os.environ.get('GNW_TAIL_CLUSTER','0')} fused={fused}: {rep.iterations} it, "
              f"{1e3*st['t_minres']:.2f} ms, {1e3*st['t_minres']/rep.iterations:.3f} ms/it", flush=True)
