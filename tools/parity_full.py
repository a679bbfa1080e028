"""Full-run parity evidence (GPU vs CPU oracle) for BASELINE configs, written to a JSON file.
usage: python tools/parity_full.py OUT.json C5[:steps] C4:20 ...
Runs the GPU path (default solver) and the oracle for the same steps and reports max |ds|,
||dc||/||c||, ||dp||/||p|| and dt agreement at the end (and the oracle / GPU wall times)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import lrbms_oracle as O  # noqa: E402
from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.lrbms import LrbmsContext  # noqa: E402

out_path = sys.argv[1]
results = []
for spec in sys.argv[2:]:
    name, _, st = spec.partition(":")
    sc = inputs.make_scenario(name)
    steps = int(st) if st else sc.n_steps
    t0 = time.time()
    ctx = LrbmsContext(sc)
    dts = ctx.run(steps, log_dt=True).cpu().numpy()
    s, p, c = (t.cpu().numpy() for t in ctx.get_state())
    t_gpu = time.time() - t0
    t0 = time.time()
    ref = O.run(sc, n_steps=steps, keep=False)
    t_cpu = time.time() - t0
    last = ref["last"]
    r = {"config": name, "steps": steps,
         "max_abs_ds": float(np.max(np.abs(s - ref["s"]))),
         "rel_dc": float(np.max(np.abs(c - last["c"])) / np.max(np.abs(last["c"]))),
         "rel_dp": float(np.max(np.abs(p - last["p"])) / np.max(np.abs(last["p"]))),
         "rel_ddt_max": float(np.max(np.abs(dts - ref["dts"]) / ref["dts"])),
         "s_range_gpu": [float(s.min()), float(s.max())],
         "oracle_seconds": t_cpu, "gpu_seconds_incl_setup": t_gpu}
    r["pass_1e-10"] = r["max_abs_ds"] <= 1e-10 and r["rel_dc"] <= 1e-10 and r["rel_dp"] <= 1e-10
    results.append(r)
    print(json.dumps(r), flush=True)
    json.dump(results, open(out_path, "w"), indent=1)
