"""Capacitance GEMM: the TMA-staged kernel (dgemm_tma.cu) against the cp.async kernel
(GNW_DGEMM_TMA=0): Cholesky factors bit for bit, and t_C of both.  Run each mode in its own
process (the switch is read once).

    python tools/check_dgemm_tma.py [C2|C4|C1|m868|n7m5 ...]
"""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def child(cfgname, out):
    import torch
    from paper_2209_02815_b200 import AmgOptions, Context, workload as W
    if cfgname.startswith("n"):  # nXXmYY: mesh n = XX (N = 2 XX^2 cells), m = YY rows
        n, m = (int(v) for v in cfgname[1:].split("m"))
        mesh = W.unit_square_mesh(n)
        ctx = Context(0)
        ctx.assemble(mesh, AmgOptions(coarse_threshold=64))
        J = W.synthetic_jacobian_device(m, mesh.n_cells, 9, "cuda")
    elif cfgname.startswith("m"):
        n, m = 128, int(cfgname[1:])
        mesh = W.unit_square_mesh(n)
        ctx = Context(0)
        ctx.assemble(mesh, AmgOptions(coarse_threshold=64))
        J = W.synthetic_jacobian_device(m, mesh.n_cells, 9, "cuda")
    else:
        cfg = W.CONFIGS[cfgname]
        inp = W.gnstep_inputs(cfg.n, cfg.m, cfg.index)
        ctx = Context(0)
        ctx.assemble(inp.mesh, AmgOptions(coarse_threshold=cfg.coarse_threshold))
        J = torch.from_numpy(inp.J).cuda()
    ctx.use_device_pointers(True)
    ts = []
    for _ in range(5):
        tm = ctx.set_jacobian(J, 1e-2)
        ts.append(tm["t_C"])
    H, L = ctx.woodbury_factors()
    np.save(out, np.asarray(L))
    print(f"{cfgname} GNW_DGEMM_TMA={os.environ.get('GNW_DGEMM_TMA', '1')}: t_C min {1e3 * min(ts):.4f} ms, launches {ctx.stats()['kernel_launches']}")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--child":
        child(sys.argv[2], sys.argv[3])
        sys.exit(0)
    for name in sys.argv[1:] or ["C2"]:
        outs = []
        for mode in ("1", "0"):
            out = f"/tmp/dgemm_{name}_{mode}.npy"
            env = dict(os.environ, GNW_DGEMM_TMA=mode)
            subprocess.run([sys.executable, __file__, "--child", name, out], env=env, check=True)
            outs.append(np.load(out))
        same = np.array_equal(outs[0], outs[1])
        print(f"{name}: Cholesky factor of C bitwise equal: {same}; max |dL| {np.abs(outs[0] - outs[1]).max():.3e}")
        assert same
