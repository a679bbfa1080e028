"""PCG iterations per step against the stopping tolerance (what the initial guess is worth, and the
convergence rate): python tools/exp_rtol_iters.py C5 pod 40"""
import json
import sys

sys.path.insert(0, ".")
from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.lrbms import LrbmsContext  # noqa: E402

cfg, basis, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
sc = inputs.make_scenario(cfg, basis=basis)
for rtol in (1e-2, 1e-4, 1e-6, 1e-8, 1e-10, 5e-13):
    for hist in (8, 0):
        ctx = LrbmsContext(sc, solver=dict(rtol=rtol, history=hist))
        ctx.run(10)
        s0 = ctx.stats()
        ctx.run(n)
        s1 = ctx.stats()
        print(json.dumps({"cfg": cfg, "rtol": rtol, "history": hist,
                          "iters_per_step": (s1["total_iters"] - s0["total_iters"]) / n}), flush=True)
        ctx.close()
