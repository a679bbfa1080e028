"""k_project phase timeline (every 8th CTA, %globaltimer) on one C5 step after warm-up."""
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
ctx.run(5)
buf = torch.zeros(1024 + 8 * 256, dtype=torch.int64, device="cuda")
ctx.L.lrbms_debug_set_tstamp.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
ctx.L.lrbms_debug_set_tstamp(ctx.h, ctypes.c_void_p(buf.data_ptr()))
ctx.stage_project()
torch.cuda.synchronize()
t = buf.cpu().numpy()[1024:].reshape(256, 8).astype(np.float64)
t = t[t[:, 0] > 0]
d = np.diff(t[:, :7], axis=1) / 1e3
names = ["issue staging", "weights", "wait Phi", "B_EE loop", "rhs+couplings", "reduction"]
print(f"{cfg}: {len(t)} CTAs sampled; CTA lifetime median {np.median((t[:, 6] - t[:, 0]) / 1e3):.2f} us")
for i, nm in enumerate(names):
    print(f"  {nm:14s} median {np.median(d[:, i]):6.2f} us  p90 {np.percentile(d[:, i], 90):6.2f}")
span = (t[:, 6].max() - t[:, 0].min()) / 1e3
print(f"  kernel span (sampled CTAs) {span:.1f} us")
