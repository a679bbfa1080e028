"""Exploration (CPU, not a test): Hestenes-Stiefel PCG vs the Chronopoulos-Gear form (one reduction
per iteration) with the A-DEF2 preconditioner and the DEF starting vector, on oracle reduced systems
(scaled: Bh = L^-1 B L^-T), fp32 coarse inverse; the CG-CG variant carries the coarse correction by
recurrence as k_pcg_tm does."""
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, ".")
from oracle import lrbms_oracle as O  # noqa: E402
from paper_1405_2810_b200 import inputs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
TRACE = len(sys.argv) > 2 and sys.argv[2] == "trace"
sc = inputs.make_scenario(cfg)
rng = np.random.default_rng(3)
s = np.clip(sc.s0 + 0.3 * rng.uniform(0, 1, sc.n), 0, 1)
lam = O.total_mobility(s, sc)
A, b = O.fine_operator(sc, lam)
blocks, r = O.project(sc, A, b)
B = O.reduced_matrix(sc, blocks).toarray()
ns, N = sc.n_s, sc.N
L = np.zeros_like(B)
for E in range(ns):
    L[E * N:(E + 1) * N, E * N:(E + 1) * N] = np.linalg.cholesky(blocks[E, 0])
Li = np.linalg.inv(L)
Bh = Li @ B @ Li.T
rb = Li @ r.reshape(-1)
zc = np.concatenate([sc.Phi[E] @ np.ones(sc.n_loc) for E in range(ns)])
Z = np.zeros((ns * N, ns))
for E in range(ns):
    Z[E * N:(E + 1) * N, E] = zc[E * N:(E + 1) * N]
Zh = L.T @ Z
Ec = Zh.T @ Bh @ Zh
Ei = np.linalg.inv(Ec).astype(np.float32).astype(np.float64)
ys = np.linalg.solve(Bh, rb)
g = lambda v: Zh.T @ (v - Bh @ v)  # noqa: E731


def hs(rtol=5e-13):
    y = Zh @ (Ei @ (Zh.T @ rb))
    res = rb - Bh @ y
    u = res + Zh @ (Ei @ g(res))
    p = u.copy(); rz = res @ u; bb = rb @ rb
    for it in range(1, 3000):
        q = Bh @ p; al = rz / (p @ q); y += al * p; res -= al * q
        u = res + Zh @ (Ei @ g(res)); rzn = res @ u
        if rzn <= rtol ** 2 * bb:
            return it, y
        p = u + rzn / rz * p; rz = rzn
    return -1, y


def cgcg(rtol=5e-13):
    y = Zh @ (Ei @ (Zh.T @ rb))
    res = rb - Bh @ y
    er = Ei @ g(res)
    u = res + Zh @ er
    bb = rb @ rb
    p = np.zeros_like(u); sv = np.zeros_like(u); es = np.zeros_like(er)
    go = ao = 1.0
    for it in range(1, 3000):
        w = Bh @ u
        ga = res @ u; de = w @ u
        if TRACE and it < 12:
            print(f"it {it}: gamma {ga:.6e} delta {de:.6e}")
        if ga <= rtol ** 2 * bb:
            return it - 1, y
        be = 0.0 if it == 1 else ga / go
        den = de if it == 1 else de - be * ga / ao
        al = ga / den
        ew = Ei @ g(w)
        p = u + be * p; sv = w + be * sv; y += al * p; res -= al * sv
        es = ew + be * es; er = er - al * es
        u = res + Zh @ er
        go, ao = ga, al
    return -1, y


for name, f in (("HS", hs), ("CG-CG", cgcg)):
    it, y = f()
    print(f"{cfg} {name}: {it} iterations, rel err {np.max(np.abs(y - ys)) / np.max(np.abs(ys)):.2e}, "
          f"true rel res {np.linalg.norm(rb - Bh @ y) / np.linalg.norm(rb):.2e}")
