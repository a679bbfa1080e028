"""On-chip PCG (k_pcg_tm, onchip=1) vs the L2-streaming PCG (k_pcg, onchip=0): same trajectory to the
parity bar, iterations and per-stage device times (CUDA events) over n steps after warm-up."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.lrbms import LrbmsContext  # noqa: E402

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2", "C3", "C4", "C5"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for cfg in cfgs:
    sc = inputs.make_scenario(cfg)
    res = {}
    for oc in (0, 1):
        ctx = LrbmsContext(sc, solver={"onchip": oc})
        ctx.run(5)
        ctx.set_profiling(True)
        s0 = ctx.stats()
        ctx.run(n)
        st = ctx.stage_times()
        s1 = ctx.stats()
        s, p, c = (t.cpu().numpy() for t in ctx.get_state())
        res[oc] = dict(s=s, c=c, iters=(s1["total_iters"] - s0["total_iters"]) / n,
                       pcg_us=1e3 * st["pcg"][0] / n, ms=sum(v[0] for v in st.values()) / n)
        ctx.close()
    dc = float(np.max(np.abs(res[0]["c"] - res[1]["c"])) / np.max(np.abs(res[0]["c"])))
    ds = float(np.max(np.abs(res[0]["s"] - res[1]["s"])))
    print(json.dumps({"cfg": cfg, "steps": n + 5, "rel_dc": dc, "abs_ds": ds,
                      "iters": [res[0]["iters"], res[1]["iters"]], "pcg_us": [round(res[0]["pcg_us"], 1), round(res[1]["pcg_us"], 1)],
                      "ms_per_step": [round(res[0]["ms"], 3), round(res[1]["ms"], 3)]}), flush=True)
