import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2209_02815_b200 import AmgOptions, Context, workload as W
cfg = W.CONFIGS["C2"]
t=time.time(); inp = W.gnstep_inputs(cfg.n, cfg.m, cfg.index); print("inputs %.1fs"%(time.time()-t), flush=True)
K, N = W.mixed_sizes(cfg.n)
t=time.time(); ctx = Context(0); ctx.assemble(inp.mesh, AmgOptions()); print("assemble %.1fs"%(time.time()-t), ctx.info(), flush=True)
for mode in ("device", "host"):
    if mode == "device":
        ctx.use_device_pointers(True)
        J = torch.from_numpy(inp.J).cuda(); dm = torch.from_numpy(inp.dm).cuda(); dg = torch.from_numpy(inp.dg).cuda()
        zN = torch.zeros(N, dtype=torch.float64, device="cuda"); zm = torch.zeros(cfg.m, dtype=torch.float64, device="cuda")
    else:
        ctx.use_device_pointers(False)
        J = torch.from_numpy(inp.J).pin_memory().numpy(); dm = inp.dm; dg = inp.dg; zN = np.zeros(N); zm = np.zeros(cfg.m)
    for k in range(6):
        a = cfg.alphas[k % 5]
        torch.cuda.synchronize()
        t0 = time.perf_counter(); tm = ctx.set_jacobian(J, a); t1 = time.perf_counter()
        b = ctx.assemble_rhs(dm, zN, dg, zm); t2 = time.perf_counter()
        x, rep = ctx.minres(b, tol=1e-8); t3 = time.perf_counter()
        st = ctx.stats()
        print(mode, a, "setJ %.1f ms (H %.1f C %.1f chol %.1f) rhs %.1f ms minres %.1f ms (dev %.1f) it %d" % (
            1e3*(t1-t0), 1e3*tm['t_H'], 1e3*tm['t_C'], 1e3*tm['t_chol'], 1e3*(t2-t1), 1e3*(t3-t2), 1e3*st['t_minres'], rep.iterations), flush=True)
