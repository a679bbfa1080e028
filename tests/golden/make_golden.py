"""Writes the oracle's C5 trajectory on the paper-recipe bases (basis = "pod") to tests/golden/.

Calls only oracle/ and the seeded input generators (paper_1405_2810_b200.inputs, whose "pod" basis is
the host offline recipe offline/recipe.py, bitwise reproducible across hosts: tools/pod_digest.py,
profiles/r02b_pod_digest.txt).  No value comes from the CUDA path.

  python tests/golden/make_golden.py [C5] [steps]

Output C5_pod_200.npz: the input digests (K, Phi), dt of every step, and at steps 10, 50 and 200 the
full saturation, the reduced coefficients and the pressure at 65536 seeded sample cells.
"""
import hashlib
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import lrbms_oracle as O  # noqa: E402
from paper_1405_2810_b200 import inputs  # noqa: E402

CHECKPOINTS = (10, 50, 200)
N_SAMPLE = 65536


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sample_cells(n):
    return np.sort(np.random.default_rng(2026).choice(n, size=min(N_SAMPLE, n), replace=False))


def main(name="C5", steps=200):
    sc = inputs.make_scenario(name)
    fp = O.fprime_max(sc)
    cells = sample_cells(sc.n)
    out = dict(name=name, steps=steps, K_sha=digest(sc.K), Phi_sha=digest(sc.Phi), cells=cells)
    s = np.array(sc.s0, np.float64)
    c = None
    dts = []
    t0 = time.time()
    for k in range(1, steps + 1):
        r = O.lrbms_step(sc, s, fpmax=fp, x0=c)
        s, c = r["s"], r["c"]
        dts.append(r["dt"])
        if k in CHECKPOINTS:
            out[f"s_{k}"] = s.copy()
            out[f"c_{k}"] = c.copy()
            out[f"p_{k}"] = r["p"][cells].copy()
        print(f"step {k} dt {r['dt']:.6e} ({time.time() - t0:.0f} s)", flush=True)
    out["dts"] = np.array(dts)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"{name}_pod_{steps}.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path))


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["C5"]), *(int(a) for a in sys.argv[2:3]))
