"""Full-run s/c parity vs the oracle for several solver settings (one oracle run per config).
usage: python tools/exp_rtol_parity.py C2 '[{"rtol":1e-12},{"rtol":3e-13}]' [steps]"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import lrbms_oracle as O  # noqa: E402
from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.lrbms import LrbmsContext  # noqa: E402

name = sys.argv[1]
settings = json.loads(sys.argv[2])
sc = inputs.make_scenario(name)
steps = int(sys.argv[3]) if len(sys.argv) > 3 else sc.n_steps
ref = O.run(sc, n_steps=steps, keep=False)
for st in settings:
    ctx = LrbmsContext(sc, solver=st)
    ctx.run(steps)
    s, p, c = (t.cpu().numpy() for t in ctx.get_state())
    info = ctx.stats()
    print(json.dumps({"cfg": name, "steps": steps, **st, "iters_per_step": info["total_iters"] / steps,
                      "max_abs_ds": float(np.max(np.abs(s - ref["s"]))),
                      "rel_dc": float(np.max(np.abs(c - ref["last"]["c"])) / np.max(np.abs(ref["last"]["c"])))}),
          flush=True)
    ctx.close()
