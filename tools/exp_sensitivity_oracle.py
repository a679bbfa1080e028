"""Round-off amplification of a configuration's trajectory, measured with the ORACLE alone:
rerun with K (1 + 1e-14 xi) and report max |ds| after the given step counts.  CPU only.
  python tools/exp_sensitivity_oracle.py C3 pod 50,100,200,500"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import lrbms_oracle as O  # noqa: E402
from paper_1405_2810_b200 import inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
basis = sys.argv[2] if len(sys.argv) > 2 else "pod"
marks = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "50,100,200,500").split(",")]


def trajectory(sc):
    fp = O.fprime_max(sc)
    s = np.array(sc.s0, np.float64)
    c = None
    out = {}
    for k in range(1, max(marks) + 1):
        r = O.lrbms_step(sc, s, fpmax=fp, x0=c)
        s, c = r["s"], r["c"]
        if k in marks:
            out[k] = s.copy()
    return out


sc = inputs.make_scenario(name, basis=basis)
a = trajectory(sc)
sc.K = sc.K * (1.0 + 1e-14 * np.random.default_rng(7).standard_normal(sc.n))
b = trajectory(sc)
print(f"{name} {basis}: max |ds| with K (1 + 1e-14 xi): " +
      ", ".join(f"{k} steps {np.max(np.abs(a[k] - b[k])):.2e}" for k in marks) +
      f"; s range after {max(marks)}: [{a[max(marks)].min():.3f}, {a[max(marks)].max():.3f}]", flush=True)
