"""Per-CTA timeline of k_pcg_tm (globaltimer stamps: loop start, before the grid reduction, after it,
after the coarse gather) on one step after warm-up: phase durations and arrival skew."""
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
buf = torch.zeros(65536 + 4 * 16 * G * 16 + 64, dtype=torch.int64, device="cuda")
ctx.L.lrbms_debug_set_tstamp.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
ctx.L.lrbms_debug_set_tstamp(ctx.h, ctypes.c_void_p(buf.data_ptr()))
ctx.run(1)
it = ctx.stats()["last_iters"]
t8 = buf.cpu().numpy()[4096:4096 + 8 * 32 * G].reshape(32, G, 8).astype(np.float64)
t = t8[:, :, :4]
g = G
rows = []
for i in range(3, min(it, 30)):
    N = (t[i, :, 1] - t[i, :, 0]) / 1e3            # phase N per CTA
    arr = (t[i, :, 1] - t[i, :, 1].min()) / 1e3      # arrival spread at the reduction
    red = (t[i, :, 2] - t[i, :, 1]) / 1e3            # reduction incl. waiting
    gat = (t[i, :, 3] - t[i, :, 2]) / 1e3            # gather + coarse products
    upd = (t[i + 1, :, 0] - t[i, :, 3]) / 1e3        # update
    exitsp = (t[i, :, 2] - t[i, :, 2].min()) / 1e3
    rows.append([np.median(N), N.max(), np.percentile(arr, 90), np.median(red), red.min(), np.percentile(exitsp, 90), np.median(gat), gat.max(),
                 np.median(upd), (t[i + 1, 0, 0] - t[i, 0, 0]) / 1e3])
r = np.median(np.array(rows), axis=0)
for i in (5, 8):
    a = (t8[i, :, 4] - t8[i, :, 1]) / 1e3   # CTA barrier (slowest warp)
    b = (t8[i, :, 5] - t8[i, :, 4]) / 1e3   # partials + red.release
    c = (t8[i, :, 6] - t8[i, :, 5]) / 1e3   # spin
    d = (t8[i, :, 2] - t8[i, :, 6]) / 1e3   # partial reads + broadcast
    lastarr = (t8[i, :, 5].max() - t8[i, :, 5].min()) / 1e3
    print(f"it {i} reduce parts med/max us: cta-bar {np.median(a):.2f}/{a.max():.2f} release {np.median(b):.2f}/{b.max():.2f}"
          f" spin {np.median(c):.2f}/{c.max():.2f} tail {np.median(d):.2f}/{d.max():.2f}; arrival (after release) spread {lastarr:.2f}")
print(f"{cfg}: G={g} iters={it}; us: N med {r[0]:.2f} max {r[1]:.2f} | arrival spread p90 {r[2]:.2f} | reduce med {r[3]:.2f}"
      f" min {r[4]:.2f} exit spread p90 {r[5]:.2f} | gather med {r[6]:.2f} max {r[7]:.2f} | update {r[8]:.2f} | iter {r[9]:.2f}")
slow = np.argsort(-(t[5, :, 1] - t[5, :, 0]))[:8]
print("slowest CTAs in phase N (it 5):", slow.tolist(), ((t[5, slow, 1] - t[5, slow, 0]) / 1e3).round(2).tolist())

w = buf.cpu().numpy()[65536:65536 + 4 * 16 * G * 16].reshape(16, G, 16, 4).astype(np.float64)
Wn = -(-sc.n_s // G)
for i in (5, 8):
    st = t[i, :, 0][:, None]
    tpass = (w[i, :, :Wn, 0] - st) / 1e3          # loop start -> T pass done
    wait = (w[i, :, :Wn, 1] - w[i, :, :Wn, 0]) / 1e3   # publish + flag wait
    upass = (w[i, :, :Wn, 2] - w[i, :, :Wn, 1]) / 1e3  # U pass
    print(f"it {i}: per-warp us  T-pass med {np.median(tpass):.2f} max {tpass.max():.2f} | wait med {np.median(wait):.2f}"
          f" max {wait.max():.2f} | U-pass med {np.median(upass):.2f} max {upass.max():.2f}")
    print("  by warp index (median over CTAs): T-pass", np.median(tpass, axis=0).round(2).tolist())
    print("  wait", np.median(wait, axis=0).round(2).tolist())
    print("  U-pass", np.median(upass, axis=0).round(2).tolist())
