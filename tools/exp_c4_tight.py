import sys
sys.path.insert(0, ".")
import numpy as np
from oracle import lrbms_oracle as O
from paper_1405_2810_b200 import inputs
from paper_1405_2810_b200.lrbms import LrbmsContext
sc = inputs.make_scenario("C4")
ref = O.run(sc, n_steps=10, keep=True)
for opts in [dict(rtol=1e-14), dict(rtol=1e-14, use_coarse=1), dict(rtol=1e-15)]:
    ctx = LrbmsContext(sc, solver=opts)
    ctx.run(10)
    s, p, c = (t.cpu().numpy() for t in ctx.get_state())
    rc = np.max(np.abs(c - ref["cs"][-1])) / np.max(np.abs(ref["cs"][-1]))
    rp = np.max(np.abs(p - ref["ps"][-1])) / np.max(np.abs(ref["ps"][-1]))
    ds = np.max(np.abs(s - ref["s"]))
    print(opts, "iters/step", ctx.stats()["total_iters"] / 10, f"rel dc {rc:.2e} dp {rp:.2e} ds {ds:.2e}", flush=True)
