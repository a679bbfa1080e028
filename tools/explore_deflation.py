"""Exploration (CPU, not a test): iteration counts of the two-level preconditioners on a reduced
system built by the oracle: additive (AD, the current one), A-DEF2 (P^T D^-1 + Q, with the DEF
starting vector) and BNN, with an exact and an fp32-rounded coarse inverse."""
import sys
import time

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, ".")
from oracle import lrbms_oracle as O  # noqa: E402
from paper_1405_2810_b200 import inputs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
t0 = time.time()
sc = inputs.make_scenario(cfg)
rng = np.random.default_rng(3)
s = np.clip(sc.s0 + 0.3 * rng.uniform(0, 1, sc.n), 0, 1)
lam = O.total_mobility(s, sc)
A, b = O.fine_operator(sc, lam)
blocks, r = O.project(sc, A, b)
B = O.reduced_matrix(sc, blocks).tocsr()
rhs = r.reshape(-1)
ns, N = sc.n_s, sc.N
Dinv = np.linalg.inv(blocks[:, 0])
print(f"{cfg}: setup {time.time() - t0:.1f}s, R = {ns * N}", flush=True)
Z = sp.csr_matrix((np.concatenate([sc.Phi[E] @ np.ones(sc.n_loc) for E in range(ns)]),
                   (np.arange(ns * N), np.repeat(np.arange(ns), N))), shape=(ns * N, ns))
Bc = (Z.T @ (B @ Z)).toarray()
Ei = np.linalg.inv(Bc)
Ei32 = Ei.astype(np.float32).astype(np.float64)
xs = sp.linalg.spsolve(B.tocsc(), rhs)


def Dj(v):
    return np.einsum("eij,ej->ei", Dinv, v.reshape(ns, N)).reshape(-1)


def run(kind, Einv, rtol=1e-12, maxit=3000, x0=None):
    Q = lambda v: Z @ (Einv @ (Z.T @ v))  # noqa: E731
    if kind == "AD":
        prec = lambda v: Dj(v) + Q(v)  # noqa: E731
    elif kind == "ADEF2":
        def prec(v):
            y = Dj(v)
            return y + Q(v - B @ y)
    else:  # BNN
        def prec(v):
            y = Q(v)
            w = v - B @ y
            t = Dj(w)
            return y + t - Q(B @ t)
    x = np.zeros_like(rhs) if x0 is None else x0.copy()
    if kind != "AD":
        x = x + Q(rhs - B @ x)
    res = rhs - B @ x
    zz = prec(res); p = zz.copy(); rz = res @ zz
    bn = np.sqrt(rhs @ prec(rhs))
    for it in range(1, maxit + 1):
        q = B @ p; al = rz / (p @ q); x += al * p; res -= al * q
        zz = prec(res); rzn = res @ zz
        if np.sqrt(abs(rzn)) <= rtol * bn:
            break
        p = zz + (rzn / rz) * p; rz = rzn
    err = np.sqrt((x - xs) @ (B @ (x - xs)) / (xs @ (B @ xs)))
    return it, err


for kind in ["AD", "ADEF2", "BNN"]:
    for nm, Ein in [("exact", Ei), ("fp32", Ei32)]:
        it, err = run(kind, Ein)
        print(f"{kind:6s} {nm:5s} iterations {it:4d}  energy error {err:.2e}", flush=True)
# warm start from a perturbed solution (mimics the history guess)
x0 = xs * (1 + 1e-4 * rng.standard_normal(xs.size))
for kind in ["AD", "ADEF2"]:
    it, err = run(kind, Ei32, x0=x0)
    print(f"warm {kind:6s} fp32 iterations {it:4d}  energy error {err:.2e}", flush=True)
# A-DEF2 without the DEF starting correction (warm start from the perturbed solution only)
def run_nostart(Einv, x0, rtol=1e-12, maxit=3000, f32=False):
    def prec(v):
        g = Z.T @ (v - B @ v)          # scaled form uses D = I; here y = D^-1 v
        y = Dj(v)
        g = Z.T @ (v - B @ y)
        if f32:
            g = g.astype(np.float32).astype(np.float64)
        return y + Z @ (Einv @ g)
    x = x0.copy(); res = rhs - B @ x
    zz = prec(res); p = zz.copy(); rz = res @ zz
    bn = np.sqrt(rhs @ prec(rhs))
    for it in range(1, maxit + 1):
        q = B @ p; al = rz / (p @ q); x += al * p; res -= al * q
        zz = prec(res); rzn = res @ zz
        if np.sqrt(abs(rzn)) <= rtol * bn:
            break
        p = zz + (rzn / rz) * p; rz = rzn
    return it, np.sqrt((x - xs) @ (B @ (x - xs)) / (xs @ (B @ xs)))
print("ADEF2 warm, no DEF start  ", run_nostart(Ei32, x0))
print("ADEF2 warm, no DEF start, fp32 coarse rhs", run_nostart(Ei32, x0, f32=True))
print("ADEF2 cold, no DEF start  ", run_nostart(Ei32, np.zeros_like(rhs)))
