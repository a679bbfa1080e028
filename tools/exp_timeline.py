"""Per-CTA timeline of k_pcg_tm (globaltimer stamps, 8 per iteration: A start, before/after the p.Bp
reduction, before/after the r.r reduction, after the coarse gather, before/after the r.z reduction)
on one step after warm-up: per-phase durations (median / max over CTAs) and arrival spreads."""
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
W = -(-sc.n_s // 148)
G = -(-sc.n_s // W)
buf = torch.zeros(4096 + 8 * 32 * G + 64, dtype=torch.int64, device="cuda")
ctx.L.lrbms_debug_set_tstamp.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
ctx.L.lrbms_debug_set_tstamp(ctx.h, ctypes.c_void_p(buf.data_ptr()))
ctx.run(1)
it = ctx.stats()["last_iters"]
t = buf.cpu().numpy()[4096:4096 + 8 * 32 * G].reshape(32, G, 8).astype(np.float64) / 1e3
names = ["A work", "pq reduce", "B work", "rr reduce", "C gather", "C work", "rz reduce"]
res = []
for i in range(3, min(it, 30)):
    d = np.diff(t[i], axis=1)       # [G, 7]
    arr = [t[i, :, k].max() - t[i, :, k].min() for k in (1, 3, 6)]
    res.append(np.concatenate([np.median(d, axis=0), d.max(axis=0), arr, [t[i + 1, 0, 0] - t[i, 0, 0]]]))
r = np.median(np.array(res), axis=0)
print(f"{cfg}: G={G} W={W} iters={it}, us per iteration {r[-1]:.2f}")
for k, n in enumerate(names):
    print(f"  {n:10s} median {r[k]:5.2f}  max {r[7 + k]:5.2f}")
print(f"  arrival spread at the reductions: pq {r[14]:.2f} rr {r[15]:.2f} rz {r[16]:.2f}")

# setup stamps (iteration-0 slots): entry, after TMEM/shared staging, before/after the history weights,
# before/after the first reduction, after the DEF start + r.z, and the loop exit
s0 = t[0]
names0 = ["staging (TMEM, smem)", "-> hist weights", "history weights", "initial guess", "bb reduction",
          "DEF start + r.z", "iterations"]
d0 = np.diff(s0[:, :8], axis=1)
print("setup phases (median / max over CTAs, us):")
for k, nm in enumerate(names0):
    print(f"  {nm:22s} {np.median(d0[:, k]):7.2f} {d0[:, k].max():7.2f}")
