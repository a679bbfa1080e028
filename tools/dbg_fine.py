import sys, numpy as np
sys.path.insert(0, ".")
from paper_1405_2810_b200 import inputs
from paper_1405_2810_b200.lrbms import LrbmsContext
from oracle import lrbms_oracle as O
for name in ["C1", "C2"]:
    sc = inputs.make_scenario(name)
    ctx = LrbmsContext(sc)
    dt, it = ctx.run_fine(1, log_dt=True, rtol=1e-14)
    s, p, _ = ctx.get_state()
    p = p.cpu().numpy(); s = s.cpu().numpy()
    po, lam = O.fine_pressure(sc, sc.s0)
    A, b = O.fine_operator(sc, lam)
    print(name, "iters", it, "rel dp", np.max(np.abs(p - po)) / np.max(np.abs(po)), "res gpu", np.linalg.norm(A @ p - b) / np.linalg.norm(b),
          "res oracle", np.linalg.norm(A @ po - b) / np.linalg.norm(b))
    d = A.diagonal()
    print(" diag", d[:5], "b", b[b != 0][:5], "nlinks", np.count_nonzero(b))
