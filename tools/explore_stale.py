"""Exploration (CPU, not a test): A-DEF2 vs additive coarse correction when the coarse inverse is
stale (built from the saturation k steps earlier), on the oracle's trajectory."""
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, ".")
from oracle import lrbms_oracle as O  # noqa: E402
from paper_1405_2810_b200 import inputs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 50
sc = inputs.make_scenario(cfg)
fp = O.fprime_max(sc)
s = np.array(sc.s0, np.float64)
ns, N = sc.n_s, sc.N


def system(s):
    lam = O.total_mobility(s, sc)
    A, b = O.fine_operator(sc, lam)
    blocks, r = O.project(sc, A, b)
    return blocks, O.reduced_matrix(sc, blocks).tocsr(), r.reshape(-1)


Z = sp.csr_matrix((np.concatenate([sc.Phi[E] @ np.ones(sc.n_loc) for E in range(ns)]),
                   (np.arange(ns * N), np.repeat(np.arange(ns), N))), shape=(ns * N, ns))
snaps = {}
for n in range(K + 1):
    if n in (0, 1, 5, 10, 25, K):
        snaps[n] = s.copy()
    out = O.lrbms_step(sc, s, fpmax=fp)
    s = out["s"]
blocks0, B0, _ = system(snaps[0])
Ei_stale = np.linalg.inv((Z.T @ (B0 @ Z)).toarray()).astype(np.float32).astype(np.float64)


def pcg(B, rhs, Dinv, Einv, kind, rtol=1e-12, maxit=2000):
    Dj = lambda v: np.einsum("eij,ej->ei", Dinv, v.reshape(ns, N)).reshape(-1)  # noqa: E731
    Q = lambda v: Z @ (Einv @ (Z.T @ v))  # noqa: E731
    if kind == "AD":
        prec = lambda v: Dj(v) + Q(v)  # noqa: E731
    elif kind == "ADEF1":
        def prec(v):
            y = Q(v)
            return y + Dj(v - B @ y)
    elif kind == "BNN":
        def prec(v):
            y = Q(v)
            w = v - B @ y
            t = Dj(w)
            return y + t - Q(B @ t)
    else:
        def prec(v):
            y = Dj(v)
            return y + Q(v - B @ y)
    x = np.zeros_like(rhs)
    if kind != "AD":
        x = x + Q(rhs - B @ x)
    res = rhs - B @ x
    zz = prec(res); p = zz.copy(); rz = res @ zz
    bn = np.linalg.norm(rhs)
    for it in range(1, maxit + 1):
        q = B @ p; al = rz / (p @ q); x += al * p; res -= al * q
        zz = prec(res); rzn = res @ zz
        if np.sqrt(abs(rzn)) <= rtol * bn:
            break
        p = zz + (rzn / rz) * p; rz = rzn
    return it


for n in sorted(snaps):
    blocks, B, rhs = system(snaps[n])
    Dinv = np.linalg.inv(blocks[:, 0])
    Ei = np.linalg.inv((Z.T @ (B @ Z)).toarray())
    print(f"step {n:3d}: AD fresh {pcg(B, rhs, Dinv, Ei, 'AD')}, AD stale {pcg(B, rhs, Dinv, Ei_stale, 'AD')}, "
          f"ADEF2 fresh {pcg(B, rhs, Dinv, Ei, 'ADEF2')}, ADEF2 stale {pcg(B, rhs, Dinv, Ei_stale, 'ADEF2')}, "
          f"BNN stale {pcg(B, rhs, Dinv, Ei_stale, 'BNN')}, ADEF1 fresh {pcg(B, rhs, Dinv, Ei, 'ADEF1')}, "
          f"ADEF1 stale {pcg(B, rhs, Dinv, Ei_stale, 'ADEF1')}",
          flush=True)
