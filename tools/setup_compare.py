"""gnw_assemble of a device context with the device AMG setup (default) and with the host setup
(GNW_DEVICE_SETUP=0), per mesh size; each mode in its own process.

    python tools/setup_compare.py 512 1024 2048
"""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
THR = {512: 64, 1024: 1024, 2048: 4096, 256: 64, 64: 64}

if len(sys.argv) > 2 and sys.argv[1] == "--child":
    from paper_2209_02815_b200 import AmgOptions, Context, workload as W
    n = int(sys.argv[2])
    Context(0)
    mesh = W.unit_square_mesh(n)
    ts = []
    for _ in range(2):
        t0 = time.time()
        c = Context(0)
        c.assemble(mesh, AmgOptions(coarse_threshold=THR.get(n, 64)))
        ts.append(time.time() - t0)
        del c
    print(f"n={n} GNW_DEVICE_SETUP={os.environ.get('GNW_DEVICE_SETUP', '1')}: assemble {min(ts):.2f} s", flush=True)
    sys.exit(0)
for n in [int(a) for a in sys.argv[1:]] or [512, 1024, 2048]:
    for mode in ("1", "0"):
        subprocess.run([sys.executable, __file__, "--child", str(n)], env=dict(os.environ, GNW_DEVICE_SETUP=mode), check=True)
