"""Host setup time (mesh, assembly, SA-AMG) per mesh size, host-only context vs a device
context (whose sparse products run on the GPU).  GNW_SETUP_TIMING=1 adds per-phase lines.

    python tools/setup_time.py [n ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_02815_b200 import AmgOptions, Context, workload as W  # noqa: E402

THR = {512: 64, 1024: 1024, 2048: 4096, 256: 64, 64: 64}
Context(0)  # CUDA context creation outside the timings
for n in [int(a) for a in sys.argv[1:]] or [512, 1024, 2048]:
    mesh = W.unit_square_mesh(n)
    for label, dev in (("host", None), ("device", 0)):
        print(f"--- n={n} {label}", file=sys.stderr, flush=True)
        t0 = time.time()
        c = Context(dev)
        c.assemble(mesh, AmgOptions(coarse_threshold=THR.get(n, 64)))
        print(f"n={n} {label:6s} setup {time.time() - t0:.2f} s", flush=True)
        del c
print("cores", os.cpu_count())
