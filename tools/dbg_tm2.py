"""Debug: progress markers of k_pcg_tm through a pinned host buffer while the solve runs."""
import ctypes
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.lrbms import LrbmsContext  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
sc = inputs.make_scenario(cfg)
ctx = LrbmsContext(sc, solver={"onchip": 1})
buf = torch.zeros(256 + 512, dtype=torch.int64).pin_memory()
ctx.L.lrbms_debug_set_tstamp.restype = None
ctx.L.lrbms_debug_set_tstamp.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
ctx.L.lrbms_debug_set_tstamp(ctx.h, buf.data_ptr())
ctx.stage_project()
torch.cuda.synchronize()
print("projected", flush=True)
done = []


def watch():
    for _ in range(40):
        time.sleep(0.5)
        if done:
            return
        print("progress", buf[256:256 + 160].tolist(), flush=True)


th = threading.Thread(target=watch, daemon=True)
th.start()
c = ctx.stage_solve()
torch.cuda.synchronize()
done.append(1)
print("solved", ctx.stats()["last_iters"], buf[256:260].tolist(), flush=True)
