"""Newton-Schulz guard over a run: PCG iterations per step in chunks, guard trips, residual maxima.
usage: python tools/exp_ns_guard.py C4 pod 41"""
import os
import sys

sys.path.insert(0, ".")
from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.lrbms import LrbmsContext  # noqa: E402

cfg, basis, chunks = sys.argv[1], sys.argv[2], int(sys.argv[3])
sc = inputs.make_scenario(cfg, basis=basis)
ctx = LrbmsContext(sc)
its, res, prev = [], [], 0
for k in range(chunks):
    ctx.run(5)
    st = ctx.stats()
    its.append((st["total_iters"] - prev) // 5)
    res.append(round(st["ns_resid_max"], 3))
    prev = st["total_iters"]
print(cfg, os.environ.get("LRBMS_LIB", "default")[-14:], "iters/step per 5-step call:", its)
print("  last-step residual per call:", res, "trips", ctx.stats()["ns_guard_trips"], "host rebuilds", ctx.stats()["coarse_rebuilds"])
