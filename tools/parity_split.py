"""Full-run parity evidence in two halves (the oracle does not need the GPU box):
  python tools/parity_split.py gpu DIR C5[:steps] ...     # on the GPU: dump s, p, c, dt per config
  python tools/parity_split.py oracle DIR OUT.json C5[:steps] ...   # on any CPU: oracle + compare
Reports max |ds|, ||dc||/||c||, ||dp||/||p|| (max norms) and the dt agreement at the end of the run."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1405_2810_b200 import inputs  # noqa: E402

mode, d = sys.argv[1], sys.argv[2]
os.makedirs(d, exist_ok=True)
if mode == "gpu":
    from paper_1405_2810_b200.lrbms import LrbmsContext
    for spec in sys.argv[3:]:
        name, _, st = spec.partition(":")
        sc = inputs.make_scenario(name)
        steps = int(st) if st else sc.n_steps
        t0 = time.time()
        ctx = LrbmsContext(sc)
        dts = ctx.run(steps, log_dt=True).cpu().numpy()
        s, p, c = (t.cpu().numpy() for t in ctx.get_state())
        np.savez(os.path.join(d, f"{name}_{steps}.npz"), s=s, p=p, c=c, dts=dts,
                 iters=ctx.stats()["total_iters"] / steps, seconds=time.time() - t0)
        print(name, steps, "done", flush=True)
else:
    from oracle import lrbms_oracle as O
    out_path = sys.argv[3]
    results = json.load(open(out_path)) if os.path.exists(out_path) else []
    for spec in sys.argv[4:]:
        name, _, st = spec.partition(":")
        sc = inputs.make_scenario(name)
        steps = int(st) if st else sc.n_steps
        g = np.load(os.path.join(d, f"{name}_{steps}.npz"))
        cache = os.path.join(d, f"oracle_{name}_{steps}.npz")   # written by this script only (calls oracle/)
        if os.path.exists(cache):
            o = np.load(cache)
            ref = {"s": o["s"], "dts": o["dts"]}
            last = {"c": o["c"], "p": o["p"]}
            t_cpu = float(o["seconds"])
        else:
            t0 = time.time()
            ref = O.run(sc, n_steps=steps, keep=False)
            t_cpu = time.time() - t0
            last = ref["last"]
            np.savez(cache, s=ref["s"], dts=ref["dts"], c=last["c"], p=last["p"], seconds=t_cpu)
        r = {"config": name, "steps": steps,
             "max_abs_ds": float(np.max(np.abs(g["s"] - ref["s"]))),
             "rel_dc": float(np.max(np.abs(g["c"] - last["c"])) / np.max(np.abs(last["c"]))),
             "rel_dp": float(np.max(np.abs(g["p"] - last["p"])) / np.max(np.abs(last["p"]))),
             "rel_ddt_max": float(np.max(np.abs(g["dts"] - ref["dts"]) / ref["dts"])),
             "s_range_gpu": [float(g["s"].min()), float(g["s"].max())],
             "gpu_pcg_iters_per_step": float(g["iters"]),
             "oracle_seconds": t_cpu, "oracle_cores": os.cpu_count(), "gpu_seconds_incl_setup": float(g["seconds"])}
        r["pass_1e-10"] = r["max_abs_ds"] <= 1e-10 and r["rel_dc"] <= 1e-10 and r["rel_dp"] <= 1e-10
        results = [x for x in results if not (x["config"] == name and x["steps"] == steps)] + [r]
        print(json.dumps(r), flush=True)
        json.dump(results, open(out_path, "w"), indent=1)
