"""Solver-accuracy / cost sweep on one GPU (self-consistency; no oracle):
run a config for its step count with several (rtol, history, coarse_refresh) settings and report
PCG iterations per step, ms per step and max |s - s_ref|, ||c - c_ref||/||c_ref|| against the
tightest setting."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.lrbms import LrbmsContext  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else None
settings = json.loads(sys.argv[3]) if len(sys.argv) > 3 else [
    {"rtol": 1e-15, "history": 0, "coarse_refresh": 1},
    {"rtol": 1e-13, "history": 1}, {"rtol": 1e-13, "history": 2}, {"rtol": 1e-13, "history": 4},
    {"rtol": 1e-13, "history": 8}, {"rtol": 1e-12, "history": 8}, {"rtol": 1e-11, "history": 8},
]
sc = inputs.make_scenario(cfg)
steps = steps or sc.n_steps
ref = None
for st in settings:
    ctx = LrbmsContext(sc, solver=st)
    torch.cuda.synchronize()
    ctx.set_profiling(True)
    t0 = time.perf_counter()
    ctx.run(steps)
    t1 = time.perf_counter()
    stg = ctx.stage_times()
    s, p, c = ctx.get_state()
    s, c = s.cpu().numpy(), c.cpu().numpy()
    info = ctx.stats()
    if ref is None:
        ref = (s, c)
    ds = float(np.max(np.abs(s - ref[0])))
    dc = float(np.max(np.abs(c - ref[1])) / np.max(np.abs(ref[1])))
    print(json.dumps({"cfg": cfg, "steps": steps, **st, "iters_per_step": info["total_iters"] / steps,
                      "ms_per_step": 1e3 * (t1 - t0) / steps, "max_ds": ds, "rel_dc": dc,
                      "pcg_ms": stg["pcg"][0] / steps, "project_ms": stg["project"][0] / steps,
                      "coarse_ms": stg["coarse"][0] / steps, "s_range": [float(s.min()), float(s.max())]}),
          flush=True)
    ctx.close()
