"""Debug: per-iteration gamma/delta of k_pcg_tm (first solve) vs the NumPy CG-CG on the oracle system."""
import ctypes
import subprocess
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import lrbms_oracle as O  # noqa: E402
from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.lrbms import LrbmsContext  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
sc = inputs.make_scenario(cfg)
rng = np.random.default_rng(3)
s = np.clip(sc.s0 + 0.3 * rng.uniform(0, 1, sc.n), 0, 1)
sc.s0 = s
for oc in (0, 1):
    ctx = LrbmsContext(sc, solver={"onchip": oc, "history": 0})
    buf = torch.zeros(1024 + 256, dtype=torch.float64, device="cuda")
    ctx.L.lrbms_debug_set_tstamp.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    ctx.L.lrbms_debug_set_tstamp(ctx.h, ctypes.c_void_p(buf.data_ptr()))
    blocks, r = ctx.stage_project()
    try:
        c = ctx.stage_solve().cpu().numpy()
    except Exception as e:
        print("error", e)
        c = None
    gd = buf.cpu().numpy()[1024:1024 + 128].reshape(64, 2)
    print("onchip", oc, "iters", ctx.stats()["last_iters"])
    if oc == 1:
        print("gamma/delta GPU:", [f"{a:.6e}/{b:.6e}" for a, b in gd[1:12]])
lam = O.total_mobility(s, sc)
A, b = O.fine_operator(sc, lam)
ob, orr = O.project(sc, A, b)
print("blocks rel diff", float(np.max(np.abs(blocks.cpu().numpy() - ob)) / np.max(np.abs(ob))))
out = subprocess.run([sys.executable, "tools/explore_cgcg.py", cfg, "trace"], capture_output=True, text=True)
print(out.stdout[-3000:])
