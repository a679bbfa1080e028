"""Measured errors of the C5 bench workload against the oracle's golden trajectory (tests/golden/C5_pod_200.npz)
after 10 and 200 steps at the default solver settings: what test_c5_golden asserts at 1e-10."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.lrbms import LrbmsContext  # noqa: E402

G = np.load("tests/golden/C5_pod_200.npz")
sc = inputs.make_scenario("C5")
for steps in (10, 200):
    ctx = LrbmsContext(sc)
    dts = ctx.run(steps, log_dt=True).cpu().numpy()
    s, p, c = (t.cpu().numpy() for t in ctx.get_state())
    rel = lambda a, b: float(np.max(np.abs(a - b)) / np.max(np.abs(b)))
    print(f"C5 {steps} steps: dt {rel(dts, G['dts'][:steps]):.2e}, c {rel(c, G[f'c_{steps}']):.2e}, "
          f"p (sampled) {rel(p[G['cells']], G[f'p_{steps}']):.2e}, |ds| {float(np.max(np.abs(s - G[f's_{steps}']))):.2e}, "
          f"PCG iterations per step {ctx.stats()['total_iters'] / steps:.1f}", flush=True)
    ctx.close()
