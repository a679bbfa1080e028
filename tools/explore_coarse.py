"""Exploration (CPU, not a test): PCG iteration counts for richer coarse spaces
(indicator only vs indicator + linear modes vs + quadratic modes) on a reduced C5-like system."""
import sys

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

sys.path.insert(0, ".")
from oracle import lrbms_oracle as O  # noqa: E402
from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.inputs import gaussian_correlated  # noqa: E402

sc = inputs.custom_scenario(64, 64, 32, 8, 8, 8, 32, seed=5, mu_o=10.0, bc="corner_columns_3d")
z = gaussian_correlated((32, 64, 64), (2.0, 16.0, 16.0), 5)
sc.K = np.exp(2.0 * z).reshape(-1)
rng = np.random.default_rng(3)
s = np.clip(rng.uniform(-0.2, 1.0, sc.n), 0, 1)          # a generic saturation field
lam = O.total_mobility(s, sc)
A, b = O.fine_operator(sc, lam)
blocks, r = O.project(sc, A, b)
B = O.reduced_matrix(sc, blocks).tocsr()
rhs = r.reshape(-1)
ns, N = sc.n_s, sc.N
Dinv = np.linalg.inv(blocks[:, 0])


def pcg(Z, rtol=1e-10, maxit=3000):
    Zs = sp.csr_matrix(Z)
    Bc = (Zs.T @ (B @ Zs)).toarray()
    cf = sla.cho_factor(Bc)
    def prec(v):
        y = np.einsum("eij,ej->ei", Dinv, v.reshape(ns, N)).reshape(-1)
        return y + Zs @ sla.cho_solve(cf, Zs.T @ v)
    x = np.zeros_like(rhs); res = rhs.copy(); zz = prec(res); p = zz.copy(); rz = res @ zz
    bn = np.sqrt(rhs @ prec(rhs))
    for it in range(1, maxit + 1):
        q = B @ p; al = rz / (p @ q); x += al * p; res -= al * q
        zz = prec(res); rzn = res @ zz
        if np.sqrt(rzn) <= rtol * bn:
            return it
        p = zz + (rzn / rz) * p; rz = rzn
    return maxit


# coarse vectors in coefficient space: Z_E[:, m] = Phi_E g_m for fine-cell functions g_m on E
lz, ly, lx = np.meshgrid(np.arange(8), np.arange(8), np.arange(8), indexing="ij")
X = ((2 * lx + 1) / 8 - 1).reshape(-1); Y = ((2 * ly + 1) / 8 - 1).reshape(-1); Zc = ((2 * lz + 1) / 8 - 1).reshape(-1)
funcs = {"1": [np.ones(512)], "1xyz": [np.ones(512), X, Y, Zc],
         "quad": [np.ones(512), X, Y, Zc, X * X, Y * Y, Zc * Zc, X * Y, X * Zc, Y * Zc]}
for name, fl in funcs.items():
    m = len(fl)
    Z = np.zeros((ns * N, ns * m))
    for E in range(ns):
        for k, gfun in enumerate(fl):
            Z[E * N:(E + 1) * N, E * m + k] = sc.Phi[E] @ gfun
    print(name, "coarse dim", ns * m, "iterations to 1e-10:", pcg(Z), flush=True)
# (block-Jacobi only needs a dedicated path; skipped)

# aggregated indicator coarse spaces (2x2x2 and 2x2x1 subdomain aggregates)
def agg_Z(ax, ay, az):
    Sx, Sy, Sz = sc.Sx, sc.Sy, sc.Sz
    na = (Sx // ax) * (Sy // ay) * (Sz // az)
    Z = np.zeros((ns * N, na))
    for E in range(ns):
        I = E % Sx; J = (E // Sx) % Sy; L = E // (Sx * Sy)
        a = I // ax + (Sx // ax) * (J // ay + (Sy // ay) * (L // az))
        Z[E * N:(E + 1) * N, a] = sc.Phi[E] @ np.ones(512)
    return Z
for agg in [(2, 2, 1), (2, 2, 2), (4, 4, 1)]:
    Z = agg_Z(*agg)
    print("aggregated", agg, "coarse dim", Z.shape[1], "iterations:", pcg(Z), flush=True)
