"""Per-stage device times (CUDA events) of a config's step over N steps after warm-up, and the true
step time (events around the whole run; stage times may overlap when the coarse update runs on the
side stream)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.lrbms import LrbmsContext  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50
affine = len(sys.argv) > 3 and sys.argv[3] == "affine"
sc = inputs.make_scenario(cfg)
ctx = LrbmsContext(sc)
if affine:
    ctx.set_profiles(inputs.profile_saturations(sc))
    ctx.set_online(True)
ctx.run(5)
s0 = ctx.stats()
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(ctx.stream)
ctx.run(n)
e1.record(ctx.stream)
torch.cuda.synchronize()
wall = e0.elapsed_time(e1) / n
s1 = ctx.stats()
ctx.set_profiling(True)
ctx.run(n)
st = ctx.stage_times()
print(json.dumps({"cfg": cfg, "ms_per_step": wall, "iters": (s1["total_iters"] - s0["total_iters"]) / n,
                  **{k: round(1e3 * v[0] / n, 1) for k, v in st.items()}}))
