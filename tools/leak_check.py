"""Device-memory leak check: repeated create / assemble / set_jacobian / solve / close cycles (device
AMG setup forced on, persistent and graph loops) must return the device's free memory to where it was."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GNW_DEVICE_SETUP", "1")
from paper_2209_02815_b200 import Context, workload as W  # noqa: E402

torch.cuda.init()
inp = W.gnstep_inputs(256, 16, 0)
free = []
for k in range(12):
    c = Context(0)
    c.assemble(inp.mesh)
    c.set_jacobian(inp.J, 1e-2)
    for mode in ("auto", "lean", "reference"):
        c.set_loop_mode(mode)
        x, rep = c.gn_step_solve(inp.dm, np.zeros(c.N), inp.dg, np.zeros(16), tol=1e-8)
        assert rep.converged
    c.close()
    torch.cuda.synchronize()
    free.append(torch.cuda.mem_get_info()[0])
    print(k, free[-1] / 1e6, "MB free", flush=True)
drift = (free[2] - free[-1]) / 1e6
print(f"free-memory drift over the last 10 cycles: {drift:.1f} MB")
assert abs(drift) < 64, drift
