"""Trajectory sensitivity measured with the GPU path itself: rerun a config with
K -> K (1 + eps xi) and report max |s - s_ref| at checkpoints (tight solver)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.lrbms import LrbmsContext  # noqa: E402

cfg = sys.argv[1]
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-14
rtol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-14
sc = inputs.make_scenario(cfg)
checkpoints = sorted(set([min(sc.n_steps, k) for k in (10, 20, 50, 100, 200, 500, 1000)]))
xi = np.random.default_rng(77).standard_normal(sc.n)
runs = []
for pert in (0.0, eps):
    sc2 = inputs.make_scenario(cfg)
    sc2.K = sc.K * (1.0 + pert * xi)
    ctx = LrbmsContext(sc2, solver={"rtol": rtol})
    snaps = {}
    done = 0
    for k in checkpoints:
        ctx.run(k - done)
        done = k
        snaps[k] = ctx.get_state()[0].cpu().numpy()
    runs.append(snaps)
out = {"cfg": cfg, "eps": eps, "rtol": rtol}
for k in checkpoints:
    out[str(k)] = float(np.max(np.abs(runs[0][k] - runs[1][k])))
print(json.dumps(out))
