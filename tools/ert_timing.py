"""t_J of the ERT configs (gnw_response_jacobian) with the device geometric MG preconditioner
and with the host SA-AMG one (GNW_ERT_PC=amg), plus their agreement.

    python tools/ert_timing.py [C4 C5]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_02815_b200 import AmgOptions, Context, workload as W  # noqa: E402

for name in (sys.argv[1:] or ["C4", "C5"]):
    ec = W.ERT_CONFIGS[name]
    e = W.ert_inputs(name)
    ctx = Context(0)
    ctx.assemble(e.mesh, AmgOptions(coarse_threshold=ec.coarse_threshold))
    ctx.set_electrodes(e.electrodes)
    ctx.use_device_pointers(True)
    model = torch.from_numpy(e.model).cuda()
    res = {}
    for pc in ("gmg", "amg"):
        os.environ["GNW_ERT_PC"] = pc
        ctx.response_jacobian(model, e.survey)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g, J, st = ctx.response_jacobian(model, e.survey)
        torch.cuda.synchronize()
        res[pc] = (time.perf_counter() - t0, g.cpu().numpy(), J, st)
        print(f"{name} {pc}: t_J {res[pc][0]:.4f} s  {st}", flush=True)
    dg = np.linalg.norm(res["gmg"][1] - res["amg"][1]) / np.linalg.norm(res["amg"][1])
    ja, jb = res["gmg"][2][:64], res["amg"][2][:64]  # first 64 rows (C5: J is 63 GB)
    dJ = (torch.linalg.norm(ja - jb) / torch.linalg.norm(jb)).item()
    print(f"{name} rel diff g {dg:.2e}  J {dJ:.2e}", flush=True)
    del res, ctx
    torch.cuda.empty_cache()
