"""Exploration (CPU, not a test): A-DEF2 with a coarse inverse kept current by one Newton-Schulz
correction per step, X <- X + X (I - E_n X), the product taken with TF32-rounded operands (10-bit
mantissa), vs the fresh inverse; along the oracle's trajectory."""
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
ns, N = sc.n_s, sc.N
Z = sp.csr_matrix((np.concatenate([sc.Phi[E] @ np.ones(sc.n_loc) for E in range(ns)]),
                   (np.arange(ns * N), np.repeat(np.arange(ns), N))), shape=(ns * N, ns))


def tf32(a):
    a = np.asarray(a, np.float32).copy()
    v = a.view(np.uint32)
    v += 0x1000          # round to nearest on the 13 dropped bits
    v &= 0xFFFFE000
    return a.astype(np.float64)


def system(s):
    lam = O.total_mobility(s, sc)
    A, b = O.fine_operator(sc, lam)
    blocks, r = O.project(sc, A, b)
    return blocks, O.reduced_matrix(sc, blocks).tocsr(), r.reshape(-1)


def pcg(B, rhs, Dinv, Einv, rtol=1e-12, maxit=2000):
    Dj = lambda v: np.einsum("eij,ej->ei", Dinv, v.reshape(ns, N)).reshape(-1)  # noqa: E731
    Q = lambda v: Z @ (Einv @ (Z.T @ v))  # noqa: E731

    def prec(v):
        y = Dj(v)
        return y + Q(v - B @ y)
    x = Q(rhs)
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


s = np.array(sc.s0, np.float64)
X = None
for n in range(K + 1):
    blocks, B, rhs = system(s)
    Ec = (Z.T @ (B @ Z)).toarray()
    if X is None:
        X = np.linalg.inv(Ec).astype(np.float32).astype(np.float64)
    else:
        R = np.eye(ns) - (Ec @ X).astype(np.float32).astype(np.float64)
        rho = np.linalg.norm(R, 2)
        X = (X + tf32(X) @ tf32(R)).astype(np.float32).astype(np.float64)
        rho2 = np.linalg.norm(np.eye(ns) - Ec @ X, 2)
        if n in (1, 2, 5, 10, 25, 50, 100, K):
            Dinv = np.linalg.inv(blocks[:, 0])
            Ei = np.linalg.inv(Ec)
            print(f"step {n:3d}: rho before {rho:.2e} after {rho2:.2e}; A-DEF2 iterations fresh "
                  f"{pcg(B, rhs, Dinv, Ei)}, NS-updated {pcg(B, rhs, Dinv, X)}", flush=True)
    s = O.lrbms_step(sc, s, fpmax=fp)["s"]
