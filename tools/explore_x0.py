"""Exploration (CPU, not a test): PCG iterations to rtol from different initial guesses over an
LRBMS trajectory -- previous solution, linear/quadratic extrapolation, Galerkin projection onto the
span of the last k solutions (B-optimal combination)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import lrbms_oracle as O  # noqa: E402
from paper_1405_2810_b200 import inputs  # noqa: E402

sc = inputs.make_scenario("C5")
# shrink C5 to a 64x64x32 grid (256 subdomains of 8x8x8), same recipe
sc2 = inputs.custom_scenario(64, 64, 32, 8, 8, 8, 32, seed=5, mu_o=10.0, bc="corner_columns_3d")
from paper_1405_2810_b200.inputs import gaussian_correlated  # noqa: E402
z = gaussian_correlated((32, 64, 64), (2.0, 16.0, 16.0), 5)
sc2.K = np.exp(2.0 * z).reshape(-1)
sc = sc2
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rtol = 1e-13
fp = O.fprime_max(sc)
s = sc.s0.copy()
hist = []
res = {k: [] for k in ["lin", "quad", "proj3", "proj6", "proj10", "proj16"]}
for n in range(steps):
    lam = O.total_mobility(s, sc)
    A, b = O.fine_operator(sc, lam)
    blocks, r = O.project(sc, A, b)
    B = O.reduced_matrix(sc, blocks)
    rv = r.reshape(-1)
    guesses = {}
    if len(hist) >= 1:
        guesses["prev"] = hist[-1]
    if len(hist) >= 2:
        guesses["lin"] = 2 * hist[-1] - hist[-2]
    if len(hist) >= 3:
        guesses["quad"] = 3 * hist[-1] - 3 * hist[-2] + hist[-3]
    for k in (3, 6, 10, 16):
        if len(hist) >= k:
            W = np.stack(hist[-k:], axis=1)
            BW = B @ W
            G = W.T @ BW
            alpha = np.linalg.lstsq(G, W.T @ rv, rcond=None)[0]
            guesses[f"proj{k}"] = W @ alpha
    c_ref = O.solve_reduced(sc, blocks, r, method="pcg")
    for name, x0 in guesses.items():
        _, it = O.solve_pcg(sc, blocks, r, x0=x0.reshape(sc.n_s, sc.N), rtol=rtol, return_iters=True)
        r0 = np.linalg.norm(rv - B @ x0) / np.linalg.norm(rv)
        res[name].append((it, r0))
    c = c_ref.reshape(-1)
    hist.append(c)
    out = O.lrbms_step(sc, s, fpmax=fp, x0=c_ref)
    s = out["s"]
    if n % 5 == 4:
        print(n, {k: (np.mean([a for a, _ in v[-5:]]), np.median([b for _, b in v[-5:]])) for k, v in res.items() if v},
              flush=True)
