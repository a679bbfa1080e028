"""Debug: one reduced solve with each PCG kernel on a small config; prints iterations and the difference."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.lrbms import LrbmsContext  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
modes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1]
sc = inputs.make_scenario(cfg)
cs = {}
for oc in modes:
    t = time.time()
    ctx = LrbmsContext(sc, solver={"onchip": oc})
    print(cfg, "onchip", oc, "created", flush=True)
    ctx.stage_project()
    c = ctx.stage_solve().cpu().numpy()
    print(cfg, "onchip", oc, "solved", ctx.stats()["last_iters"], f"{time.time() - t:.1f}s", flush=True)
    cs[oc] = c
    ctx.run(3)
    print(cfg, "onchip", oc, "ran 3 steps", ctx.stats()["total_iters"], flush=True)
if len(cs) == 2:
    print("rel dc", float(np.max(np.abs(cs[0] - cs[1])) / np.max(np.abs(cs[0]))))
