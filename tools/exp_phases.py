"""PCG phase timing (CTA 0 %globaltimer stamps) on one C5 step after warm-up."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.lrbms import LrbmsContext  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
sc = inputs.make_scenario(cfg)
ctx = LrbmsContext(sc)
ctx.run(10)
buf = torch.zeros(256 + 8 * 64, dtype=torch.int64, device="cuda")
ctx.L.lrbms_debug_set_tstamp.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
ctx.L.lrbms_debug_set_tstamp(ctx.h, ctypes.c_void_p(buf.data_ptr()))
ctx.run(1)
full = buf.cpu().numpy().astype(np.float64)
t = full[:256].reshape(64, 4)
f = full[256:].reshape(64, 8)
it = ctx.stats()["last_iters"]
rows = []
for i in range(2, min(it, 60)):
    a = t[i, 0] - t[i - 1, 3]   # phase A work (after previous sync C) until before sync
    sa = t[i, 1] - t[i, 0]      # sync A (incl. partial)
    b = t[i, 2] - t[i, 1]       # phase B + sync B
    c = t[i, 3] - t[i, 2]       # phase C + sync C
    rows.append((a, sa, b, c))
r = np.median(np.array(rows), axis=0) / 1e3
print(f"iters {it}: median us  A-work {r[0]:.2f}  A-sync {r[1]:.2f}  B(work+sync) {r[2]:.2f}  C(work+sync) {r[3]:.2f}"
      f"  total {r.sum():.2f}")

