"""Per-stage device times (CUDA events) of the C5 step over N steps after warm-up."""
import json
import sys

sys.path.insert(0, ".")
from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.lrbms import LrbmsContext  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50
sc = inputs.make_scenario(cfg)
ctx = LrbmsContext(sc)
ctx.run(5)
ctx.set_profiling(True)
s0 = ctx.stats()
ctx.run(n)
st = ctx.stage_times()
s1 = ctx.stats()
tot = sum(v[0] for v in st.values())
print(json.dumps({"cfg": cfg, "ms_per_step": tot / n, "iters": (s1["total_iters"] - s0["total_iters"]) / n,
                  **{k: round(1e3 * v[0] / n, 1) for k, v in st.items()}}))
