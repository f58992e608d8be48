"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize_case.py

* a C1-shaped GN step (n = 32, m = 16) on every loop schedule, through the conditional-WHILE
  graph (last-block atomics, PDL launch_dependents / wait pairs, device-selected ring slots);
* the same solve with GNW_NO_GRAPH semantics is not needed: the graph body is the same kernels;
* a LocalComm P = 2 partitioned solve (cross-thread device buffers, host barriers).
Prints one line per case; exits non-zero on any solver error."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2209_02815_b200 import Context, run_ranks, workload as W  # noqa: E402


def main():
    n, m, alpha = 32, 16, 1e-2
    inp = W.gnstep_inputs(n, m, 0)
    c = Context(0)
    c.assemble(inp.mesh)
    c.set_jacobian(inp.J, alpha)
    b = c.assemble_rhs(inp.dm, np.zeros(c.N), inp.dg, np.zeros(m))
    for mode in ("reference", "fused", "lean"):
        c.set_loop_mode(mode)
        x, rep = c.minres(b, tol=1e-8)
        print(f"single {mode}: {rep.iterations} iterations, converged {rep.converged}", flush=True)
    c.set_coarse_mode(True)
    x, rep = c.minres(b, tol=1e-8)
    print(f"single exact coarse: {rep.iterations} iterations", flush=True)
    c.close()

    ctxs = Context.local_group(2)

    def body(ctx, r):
        ctx.assemble(inp.mesh)
        p = ctx.partition()
        ctx.set_jacobian(np.ascontiguousarray(inp.J[:, p["c_lo"]:p["c_hi"]]), alpha)
        bb = ctx.assemble_rhs(inp.dm, np.zeros(ctx.N), inp.dg, np.zeros(m))
        return ctx.minres(bb, tol=1e-8)[1].iterations

    print("local group P=2:", run_ranks(ctxs, body), flush=True)


if __name__ == "__main__":
    main()
