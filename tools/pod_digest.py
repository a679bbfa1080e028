"""Digests of the seeded inputs and of the host offline recipe's bases (basis = "pod") per config:
checks that the recipe is bitwise reproducible across hosts (this container vs the GPU box)."""
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1405_2810_b200 import inputs  # noqa: E402


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


for name in (sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]):
    t = time.time()
    sc = inputs.make_scenario(name)
    print(f"{name}: K {h(sc.K)} Phi {h(sc.Phi)} ({time.time() - t:.1f} s, {os.cpu_count()} cpus)", flush=True)
