"""Offline basis recipe of LRBMS on the host (``basis = "pod"``): the local reduced bases Phi_E.

An INPUT GENERATOR, like ``paper_1405_2810_b200/inputs.py``: the bases are a shared input of the
online step (BASELINE.json north_star: "the offline stage ... may run on the host; its bases are
shared inputs, not the benchmarked path").  This module is neither the oracle (``oracle/``) nor the
library (``liblrbms.so``): it imports neither and neither imports it.  Tests and ``bench.py`` call
it to build Phi; the GPU offline stage (NEXT-3, ``lrbms_offline_*``) is checked against it.

It follows the initialisation of alg:lrbmsBasisConstruction, the training set
of P:663-670 / P:1026-1028, the fine snapshots of P:679-680 and the data compression
(PCA) of P:706-719 with the coarse unit functions of P:1110-1111, in the paper's order:

  1. fine pressure and velocity at s = S0 (def:pressureDG P:337-345 at k = 0, R2);
  2. time of flight (eq:timeOfFlight P:505-512 at k = 0: upwind DG0, solved cell by cell in
     descending-pressure order -- the flow-ordered back-substitution of P:517-521);
  3. M mobility profiles lambda_{alpha,q} with the horizon T = n_steps * dt^0 (A31);
  4. 2N training parameters mu in the simplex (normalised exponentials clamped at 1e-4);
  5. fine snapshots p(lambda^(j)), lambda_alpha^(j) = sum_q mu_q lambda_{alpha,q};
  6. per subdomain: the snapshot restrictions with the normalised indicator v0 projected out, their
     thin SVD (POD without mean subtraction), Phi_E = [v0, leading left singular vectors]
     (P:706-719); modes below the noise floor are not kept, and a rank-deficient Phi_E
     is completed by graded monomials orthogonalised against it (reading A32).

fp64 NumPy/SciPy.  Fine solves: sparse LU (SuperLU) up to 300k cells; above, a two-level PCG
(Jacobi + subdomain-indicator coarse space) to a relative residual of 1e-14, snapshots in parallel
worker processes (single-threaded each, so the result does not depend on the core count).
"""
from __future__ import annotations

import dataclasses
import os
from typing import Optional

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

DIRECT_MAX_CELLS = 300_000
PARALLEL_MIN_CELLS = 50_000     # snapshots of larger problems are solved in worker processes


# ----------------------------------------------------------------------------- mobilities (R5)

def phase_mobilities(sc, s):
    """lambda_w = S_e^nw / mu_w, lambda_o = (1 - S_e)^no / mu_o, S_e clamped to [0, 1] (eq:brooksCorey
    P:183-186 with the Corey law of reading R5)."""
    se = np.clip((np.asarray(s, np.float64) - sc.swr) / (1.0 - sc.swr - sc.sor), 0.0, 1.0)
    return se ** sc.nw / sc.mu_w, (1.0 - se) ** sc.no / sc.mu_o


def max_wave_speed(sc, samples=20_001):
    """max over the mobile range of d f_w / d s (sets the profile horizon T through dt^0): the
    derivative of f_w = a/(a + b), a = S_e^nw/mu_w, b = (1 - S_e)^no/mu_o, sampled on a uniform grid,
    then refined by golden-section search around the best sample."""
    def fprime(se):
        se = np.asarray(se, np.float64)
        a = se ** sc.nw / sc.mu_w
        b = (1.0 - se) ** sc.no / sc.mu_o
        da = sc.nw * se ** (sc.nw - 1.0) / sc.mu_w
        db = -sc.no * (1.0 - se) ** (sc.no - 1.0) / sc.mu_o
        return (da * b - a * db) / (a + b) ** 2
    xs = np.linspace(0.0, 1.0, samples)
    v = fprime(xs)
    k = int(np.argmax(v))
    lo, hi = xs[max(k - 1, 0)], xs[min(k + 1, samples - 1)]
    gr = (np.sqrt(5.0) - 1.0) / 2.0
    for _ in range(200):
        c1 = hi - gr * (hi - lo)
        c2 = lo + gr * (hi - lo)
        if fprime(c1) >= fprime(c2):
            hi = c2
        else:
            lo = c1
        if hi - lo < 1e-15:
            break
    best = max(float(fprime(0.5 * (lo + hi))), float(v[k]))
    return best / (1.0 - sc.swr - sc.sor)


# ----------------------------------------------------------------------------- fine k = 0 system

def _faces(sc):
    """(a, b, |F|/d_F) of the interior faces, axis by axis (cells x fastest)."""
    nx, ny, nz = sc.nx, sc.ny, sc.nz
    h = (sc.hx, sc.hy, sc.hz)
    idx = np.arange(sc.n).reshape(nz, ny, nx)
    out = []
    for ax, (sl_a, sl_b) in enumerate([((slice(None), slice(None), slice(0, -1)), (slice(None), slice(None), slice(1, None))),
                                       ((slice(None), slice(0, -1), slice(None)), (slice(None), slice(1, None), slice(None))),
                                       ((slice(0, -1), slice(None), slice(None)), (slice(1, None), slice(None), slice(None)))]):
        if (nx, ny, nz)[ax] < 2:
            continue
        a = idx[sl_a].reshape(-1)
        b = idx[sl_b].reshape(-1)
        geo = h[(ax + 1) % 3] * h[(ax + 2) % 3] / h[ax]
        out.append((a, b, np.full(a.shape, geo)))
    if not out:
        e = np.zeros(0, np.int64)
        return e, e, np.zeros(0)
    return tuple(np.concatenate(z) for z in zip(*out))


def fine_system(sc, lam):
    """A(lambda), b(lambda) of def:pressureDG at k = 0 with the lambda-weighted SWIP penalty (R2):
    w_F = |F|/d_F * 2 K_a K_b/(K_a + K_b) * (tau_a lambda_a + tau_b lambda_b), tau = K/(K_a + K_b);
    links g_L = 2 |F|/h K_a lambda_a to p_L (R6).  Returns (A csr, b, (a, b, w), (cell, g))."""
    K = sc.K
    a, b, geo = _faces(sc)
    ka, kb = K[a], K[b]
    w = geo * 2.0 * ka * kb / (ka + kb) * (ka * lam[a] + kb * lam[b]) / (ka + kb)
    h = (sc.hx, sc.hy, sc.hz)
    lc = np.asarray(sc.link_cell, np.int64)
    lgeo = np.array([2.0 * h[(d + 1) % 3] * h[(d + 2) % 3] / h[d] for d in range(3)])[np.asarray(sc.link_axis)]
    g = lgeo * K[lc] * lam[lc]
    n = sc.n
    diag = np.zeros(n)
    np.add.at(diag, a, w)
    np.add.at(diag, b, w)
    np.add.at(diag, lc, g)
    A = sp.csr_matrix((np.concatenate([diag, -w, -w]),
                       (np.concatenate([np.arange(n), a, b]), np.concatenate([np.arange(n), b, a]))), shape=(n, n))
    rhs = np.zeros(n)
    np.add.at(rhs, lc, g * np.asarray(sc.link_p))
    return A, rhs, (a, b, w), (lc, g)


def _subdomain_of_cell(sc):
    i = np.arange(sc.n)
    x, y, z = i % sc.nx, (i // sc.nx) % sc.ny, i // (sc.nx * sc.ny)
    return (x // sc.sx) + sc.Sx * ((y // sc.sy) + sc.Sy * (z // sc.sz))


def _pcg_two_level(A, rhs, sub, n_s, x0=None, rtol=1e-14, maxiter=20000):
    """CG preconditioned by Jacobi + an additive coarse correction on the subdomain indicators
    (E = Z^T A Z, dense Cholesky).  Plain loops, fixed operation order."""
    n = A.shape[0]
    d = A.diagonal()
    Z = sp.csr_matrix((np.ones(n), (np.arange(n), sub)), shape=(n, n_s))
    E = (Z.T @ (A @ Z)).toarray()
    cf = sla.cho_factor(E, lower=True)

    def prec(r):
        return r / d + Z @ sla.cho_solve(cf, Z.T @ r)

    x = np.zeros(n) if x0 is None else x0.copy()
    r = rhs - A @ x
    z = prec(r)
    p = z.copy()
    rz = float(r @ z)
    bn = float(np.linalg.norm(rhs))
    for it in range(1, maxiter + 1):
        q = A @ p
        al = rz / float(p @ q)
        x += al * p
        r -= al * q
        if float(np.linalg.norm(r)) <= rtol * bn:
            return x, it
        z = prec(r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    raise RuntimeError(f"offline fine PCG did not reach rtol {rtol} in {maxiter} iterations")


def fine_solve(sc, lam, x0=None):
    """Fine pressure of def:pressureDG for the mobility field lam."""
    A, rhs, _, _ = fine_system(sc, lam)
    if sc.n <= DIRECT_MAX_CELLS:
        return spla.splu(A.tocsc()).solve(rhs)
    return _pcg_two_level(A, rhs, _subdomain_of_cell(sc), sc.n_s, x0=x0)[0]


# ----------------------------------------------------------------------------- step 1: initial flow

def initial_flow(sc):
    """Pressure, face/link fluxes and the CFL step at s = S0 (alg:lrbmsBasisConstruction step 1(a),
    P:644-646; fluxes of eq:velocityDG at k = 0, reading R4 for dt^0)."""
    lw, lo = phase_mobilities(sc, sc.s0)
    lam = lw + lo
    p = fine_solve(sc, lam)
    A, rhs, (a, b, w), (lc, g) = fine_system(sc, lam)
    Ff = w * (p[a] - p[b])
    Fl = g * (p[lc] - np.asarray(sc.link_p))
    out = np.zeros(sc.n)
    inn = np.zeros(sc.n)
    np.add.at(out, a, np.maximum(Ff, 0)); np.add.at(inn, a, np.maximum(-Ff, 0))
    np.add.at(out, b, np.maximum(-Ff, 0)); np.add.at(inn, b, np.maximum(Ff, 0))
    np.add.at(out, lc, np.maximum(Fl, 0)); np.add.at(inn, lc, np.maximum(-Fl, 0))
    Q = np.maximum(out, inn)
    phiV = (np.ones(sc.n) if sc.phi is None else sc.phi) * sc.hx * sc.hy * sc.hz
    m = Q > 0
    dt0 = float(sc.cfl * np.min(phiV[m] / (max_wave_speed(sc) * Q[m])))
    return dict(p=p, Ff=Ff, Fl=Fl, faces=(a, b), link_cells=lc, dt0=dt0, phiV=phiV)


# ----------------------------------------------------------------------------- step 2: time of flight

def time_of_flight(sc, p, faces, Ff, link_cells, Fl, phiV):
    """DG0 upwind discretisation of eq:timeOfFlight: per cell T,
        tau_T * sum_{F out of T} |u.n|_F  =  int_T phi  +  sum_{F into T} |u.n|_F tau_up(F),
    tau_up = 0 across inflow boundary links (the particle starts on the inflow boundary).
    TPFA fluxes run from high to low pressure, so visiting cells in descending-pressure order is the
    lower block-triangular back-substitution of P:517-521 (equal pressures carry no flux).  Cells
    with no outflow (stagnant) get the largest finite tau (reading)."""
    a, b = faces
    n = sc.n
    out_sum = np.zeros(n)
    np.add.at(out_sum, a, np.maximum(Ff, 0)); np.add.at(out_sum, b, np.maximum(-Ff, 0))
    np.add.at(out_sum, link_cells, np.maximum(Fl, 0))
    # inflow lists per cell: (upwind cell, |F|) over interior faces
    up = np.where(Ff > 0, a, b)
    dn = np.where(Ff > 0, b, a)
    mag = np.abs(Ff)
    keep = mag > 0
    up, dn, mag = up[keep], dn[keep], mag[keep]
    order_in = np.argsort(dn, kind="stable")
    dn_s, up_s, mag_s = dn[order_in], up[order_in], mag[order_in]
    ptr = np.searchsorted(dn_s, np.arange(n + 1))
    order = np.argsort(-p, kind="stable")
    tau = np.full(n, np.nan)
    phiV_l, out_l, ptr_l = phiV.tolist(), out_sum.tolist(), ptr.tolist()
    up_l, mag_l = up_s.tolist(), mag_s.tolist()
    tau_l = [float("nan")] * n
    for i in order.tolist():
        o = out_l[i]
        if o <= 0.0:
            continue
        acc = phiV_l[i]
        for k in range(ptr_l[i], ptr_l[i + 1]):
            acc += mag_l[k] * tau_l[up_l[k]]
        tau_l[i] = acc / o
    tau = np.array(tau_l)
    finite = np.isfinite(tau)
    if not np.any(finite):
        raise ValueError("time of flight: no flow")
    tau[~finite] = np.max(tau[finite])
    return tau


def tof_matrix(sc, faces, Ff, link_cells, Fl, phiV):
    """The same DG0 time-of-flight system as one sparse matrix (for the monolithic-solve pin)."""
    a, b = faces
    n = sc.n
    out_sum = np.zeros(n)
    np.add.at(out_sum, a, np.maximum(Ff, 0)); np.add.at(out_sum, b, np.maximum(-Ff, 0))
    np.add.at(out_sum, link_cells, np.maximum(Fl, 0))
    up = np.where(Ff > 0, a, b)
    dn = np.where(Ff > 0, b, a)
    M = sp.csr_matrix((np.concatenate([out_sum, -np.abs(Ff)]),
                       (np.concatenate([np.arange(n), dn]), np.concatenate([np.arange(n), up]))), shape=(n, n))
    return M, phiV


# ----------------------------------------------------------------------------- step 3: mobility profiles

def mobility_profiles(sc, tau, T, M=8, s_inj=1.0):
    """lambda_{alpha,q} of P:650-662: q = 1 the mobility of S0 everywhere, q = M that of the injected
    saturation, q = 2..M-1 the S0 mobility where tau > (q-1) T/(M-2) and the injected one otherwise.
    (P:650-662 writes lambda_alpha(0) / lambda_alpha(1), i.e. S0 = 0 and S_inj = 1 of the paper's
    setup; the figure caption's index 0 is read as q = 1, A21.)  Returns (lam_w [M][n], lam_o [M][n])."""
    lw0, lo0 = phase_mobilities(sc, np.asarray(sc.s0, np.float64))
    lw1, lo1 = phase_mobilities(sc, np.full(sc.n, s_inj))
    LW = np.empty((M, sc.n))
    LO = np.empty((M, sc.n))
    for q in range(1, M + 1):
        if q == 1:
            inj = np.zeros(sc.n, bool)
        elif q == M:
            inj = np.ones(sc.n, bool)
        else:
            inj = ~(tau > (q - 1) * T / (M - 2))
        LW[q - 1] = np.where(inj, lw1, lw0)
        LO[q - 1] = np.where(inj, lo1, lo0)
    return LW, LO


# ----------------------------------------------------------------------------- step 4: training set

def training_parameters(M, count, seed):
    """count parameters mu in the simplex {mu_q >= 1e-4, sum mu_q = 1}: normalised
    exponentials (uniform on the simplex), entries clamped to >= 1e-4, renormalised."""
    rng = np.random.default_rng(seed)
    e = rng.exponential(size=(count, M))
    mu = e / e.sum(axis=1, keepdims=True)
    mu = np.maximum(mu, 1e-4)
    return mu / mu.sum(axis=1, keepdims=True)


# ----------------------------------------------------------------------------- step 5: snapshots

_WORK = {}


def _snapshot_worker(j):
    from threadpoolctl import threadpool_limits
    sc, lam, p0 = _WORK["sc"], _WORK["lam"][j], _WORK["p0"]
    with threadpool_limits(1):
        return j, fine_solve(sc, lam, x0=p0)


def snapshots(sc, LW, LO, mus, p0=None, workers=None):
    """p(lambda^(j)) for lambda_alpha^(j) = sum_q mu_q lambda_{alpha,q}: the fine solve
    with total mobility lambda_w^(j) + lambda_o^(j).  Returns [n_train][n]."""
    lam = mus @ (LW + LO)
    P = np.empty((len(mus), sc.n))
    if sc.n <= PARALLEL_MIN_CELLS:
        for j in range(len(mus)):
            P[j] = fine_solve(sc, lam[j])
        return P
    import multiprocessing as mp
    _WORK.update(sc=sc, lam=lam, p0=p0)
    workers = workers or min(len(mus), os.cpu_count() or 1)
    with mp.get_context("fork").Pool(workers) as pool:
        for j, pj in pool.imap_unordered(_snapshot_worker, range(len(mus))):
            P[j] = pj
    _WORK.clear()
    return P


# ----------------------------------------------------------------------------- step 6: per-E POD

def _graded_monomials(sc, count):
    lz, ly, lx = np.meshgrid(np.arange(sc.sz), np.arange(sc.sy), np.arange(sc.sx), indexing="ij")
    X = (2 * lx.reshape(-1) + 1) / sc.sx - 1.0
    Y = (2 * ly.reshape(-1) + 1) / sc.sy - 1.0
    Z = (2 * lz.reshape(-1) + 1) / max(sc.sz, 1) - 1.0
    cols, deg = [], 0
    while len(cols) < count and deg <= 64:
        for ez in range(deg + 1 if sc.dim == 3 else 1):
            for ey in range(deg - ez + 1):
                cols.append(X ** (deg - ey - ez) * Y ** ey * Z ** ez)
        deg += 1
    return np.stack(cols, axis=1)


def local_cells(sc):
    """cells[E, l]: fine cell of local cell l = lx + sx (ly + sy lz) in subdomain E."""
    L, J, I = np.meshgrid(np.arange(sc.Sz), np.arange(sc.Sy), np.arange(sc.Sx), indexing="ij")
    lz, ly, lx = np.meshgrid(np.arange(sc.sz), np.arange(sc.sy), np.arange(sc.sx), indexing="ij")
    I, J, L = I.reshape(-1, 1), J.reshape(-1, 1), L.reshape(-1, 1)
    return ((I * sc.sx + lx.reshape(1, -1)) + sc.nx * ((J * sc.sy + ly.reshape(1, -1))
                                                       + sc.ny * (L * sc.sz + lz.reshape(1, -1))))


def pod_bases(sc, P, N, eps_pca=1e-8):
    """Phi_E = [v0, U_1..U_{N-1}] per subdomain:
    Y_E = (I - v0 v0^T) P|_E (snapshots as columns), thin SVD without mean subtraction, left
    singular vectors in decreasing singular value, each signed so that its largest-magnitude entry
    is positive.  A mode is kept if sigma > eps_pca * sigma_ref, sigma_ref the largest Y_E singular
    value over all subdomains (the snapshots' noise floor is global).  If fewer than N - 1 modes
    remain, Phi_E is completed by graded monomials orthogonalised against it (A32).
    Returns (Phi [n_s][N][n_loc], kept [n_s]: POD modes kept per subdomain)."""
    nl = sc.n_loc
    v0 = np.full(nl, 1.0 / np.sqrt(nl))
    cells = local_cells(sc)
    Y = P.T[cells]                                   # [n_s][n_loc][n_train]
    Y = Y - v0[None, :, None] * np.einsum("l,elj->ej", v0, Y)[:, None, :]
    U, S, _ = np.linalg.svd(Y, full_matrices=False)  # batched LAPACK gesdd
    sref = float(np.max(S[:, 0])) if S.size else 0.0
    mono = _graded_monomials(sc, N + 8)
    Phi = np.empty((sc.n_s, N, nl))
    kept = np.zeros(sc.n_s, np.int64)
    for E in range(sc.n_s):
        k = int(min(N - 1, np.sum(S[E] > eps_pca * sref)))
        Q = v0[:, None]
        # the kept modes, then the monomials, each orthogonalised against the columns before it
        # (classical Gram-Schmidt, twice): the modes' v0 component is at rounding level relative to
        # sigma_1, i.e. up to eps sigma_1 / sigma_k relative to themselves
        cands = [(U[E, :, m], 0.5) for m in range(k)] + [(c, 1e-8) for c in mono.T]
        for c, tol in cands:
            if Q.shape[1] == N:
                break
            v = c.copy()
            for _ in range(2):
                v -= Q @ (Q.T @ v)
            nv = np.linalg.norm(v)
            if nv > tol * np.linalg.norm(c):
                v = v / nv
                v = v * (1.0 if v[np.argmax(np.abs(v))] > 0 else -1.0)
                Q = np.concatenate([Q, v[:, None]], axis=1)
        if Q.shape[1] < N:
            raise ValueError(f"pod basis: subdomain {E} cannot be completed to N = {N}")
        Phi[E] = Q.T
        kept[E] = k
    return Phi, kept, S


# ----------------------------------------------------------------------------- greedy basis extension

def _block_basis(sc, cols, cells):
    """The global reduced basis as a sparse n x R matrix: column (E, k) holds local function k of E."""
    rows, cidx, vals, off = [], [], [], 0
    for E in range(sc.n_s):
        Q = cols[E]
        m = Q.shape[1]
        rows.append(np.repeat(cells[E], m))
        cidx.append(np.tile(off + np.arange(m), len(cells[E])))
        vals.append(Q.reshape(-1))
        off += m
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cidx))), shape=(sc.n, off))


def greedy_bases(sc, P, LAM, N, lam_bar, eps_tol=0.0, eps_rel=1e-10, complete=True):
    """The basis extension of alg:lrbmsBasisConstruction with the paper's error measure of the
    experiments, the TRUE error in the energy norm of a fixed mobility lam_bar:
        err(mu) = [ a(p_H(mu) - p_h(mu), p_H(mu) - p_h(mu); lam_bar) ]^(1/2).
    P [J][n]: the fine pressures p_h of the training mobilities LAM [J][n] (the strong greedy needs them
    all).  The local bases start from the coarse unit function v0 = 1/sqrt(n_loc) (A15);
    every round solves the reduced problem (def:coarseScalePressure) of every training mobility in the
    current space, picks the worst approximated one, and extends every local basis by the Gram-Schmidt
    orthonormalisation of that snapshot's restriction (dependent restrictions are skipped, so the local
    sizes may differ).  Stops when the largest error is <= max(eps_tol, eps_rel x the first round's largest
    error), when a local basis reaches N (the ABI's fixed size), or when every snapshot has been used.  complete: bases shorter than N are completed by
    graded monomials (A32).  Returns (Phi [n_s][N][n_loc] or the ragged list, sizes [n_s], selected
    indices, the history of (max error, argmax) per round, the last round's errors)."""
    J = P.shape[0]
    cells = local_cells(sc)
    nl = sc.n_loc
    v0 = np.full(nl, 1.0 / np.sqrt(nl))
    cols = [v0[:, None].copy() for _ in range(sc.n_s)]
    systems = [fine_system(sc, LAM[j])[:2] for j in range(J)]
    A_bar = fine_system(sc, lam_bar)[0]
    selected, history = [], []
    err = np.zeros(J)
    while True:
        Z = _block_basis(sc, cols, cells)
        for j in range(J):
            A, b = systems[j]
            B = (Z.T @ (A @ Z)).tocsc()
            c = spla.spsolve(B, Z.T @ b)
            e = Z @ np.atleast_1d(c) - P[j]
            err[j] = float(np.sqrt(max(e @ (A_bar @ e), 0.0)))
        jmax = int(np.argmax(err))
        history.append((float(err[jmax]), jmax))
        if err[jmax] <= max(eps_tol, eps_rel * history[0][0]) or len(selected) == J or max(q.shape[1] for q in cols) >= N:
            break
        if jmax in selected:      # its restrictions were all dependent: nothing left to add for it
            break
        selected.append(jmax)
        for E in range(sc.n_s):
            v = P[jmax][cells[E]].copy()
            nv0 = np.linalg.norm(v)
            for _ in range(2):
                v -= cols[E] @ (cols[E].T @ v)
            nv = np.linalg.norm(v)
            if nv > 1e-10 * nv0 and cols[E].shape[1] < N:
                v /= nv
                v *= 1.0 if v[np.argmax(np.abs(v))] > 0 else -1.0
                cols[E] = np.concatenate([cols[E], v[:, None]], axis=1)
    sizes = np.array([q.shape[1] for q in cols])
    if not complete:
        return cols, sizes, selected, history, err.copy()
    mono = _graded_monomials(sc, N + 8)
    Phi = np.empty((sc.n_s, N, nl))
    for E in range(sc.n_s):
        Q = cols[E]
        for c in mono.T:
            if Q.shape[1] == N:
                break
            v = c.copy()
            for _ in range(2):
                v -= Q @ (Q.T @ v)
            nv = np.linalg.norm(v)
            if nv > 1e-8 * np.linalg.norm(c):
                v = v / nv
                v = v * (1.0 if v[np.argmax(np.abs(v))] > 0 else -1.0)
                Q = np.concatenate([Q, v[:, None]], axis=1)
        if Q.shape[1] < N:
            raise ValueError(f"greedy basis: subdomain {E} cannot be completed to N = {N}")
        Phi[E] = Q.T
    return Phi, sizes, selected, history, err.copy()


def greedy_recipe(sc, seed, M=8, n_train=None, eps_tol=0.0, workers=None):
    """The offline recipe with the greedy extension instead of the POD of all snapshots: steps 1-5 of
    the module header, then ``greedy_bases`` with lam_bar the mobility of the barycentre parameter
    (mu_q = 1/M).  For the configurations whose reduced problems a sparse direct solver handles in
    seconds (C1-C3)."""
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        N = sc.N
        n_train = 2 * N if n_train is None else n_train
        fl = initial_flow(sc)
        tau = time_of_flight(sc, fl["p"], fl["faces"], fl["Ff"], fl["link_cells"], fl["Fl"], fl["phiV"])
        T = sc.n_steps * fl["dt0"]
        LW, LO = mobility_profiles(sc, tau, T, M=M, s_inj=float(np.max(sc.link_s)))
        mus = training_parameters(M, n_train, seed)
        P = snapshots(sc, LW, LO, mus, p0=fl["p"], workers=workers)
        LAM = mus @ (LW + LO)
        lam_bar = np.full(M, 1.0 / M) @ (LW + LO)
        Phi, sizes, selected, history, err = greedy_bases(sc, P, LAM, N, lam_bar, eps_tol=eps_tol)
    return dict(Phi=Phi, sizes=sizes, selected=selected, history=history, errors=err, mus=mus, P=P, LAM=LAM,
                lam_bar=lam_bar)


# ----------------------------------------------------------------------------- the recipe

@dataclasses.dataclass
class OfflineResult:
    Phi: np.ndarray
    kept: np.ndarray
    sigma: np.ndarray
    tau: np.ndarray
    T: float
    dt0: float
    mus: np.ndarray
    LW: np.ndarray
    LO: np.ndarray
    P: Optional[np.ndarray] = None


def pod_recipe(sc, seed, M=8, n_train=None, keep_snapshots=False, workers=None, eps_pca=1e-8):
    """The whole offline recipe for scenario ``sc`` (its K, links, s0, N, n_steps): steps 1-6 above.
    seed: training-set seed (100 + config index for C1..C5)."""
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):   # BLAS reductions in a fixed order: bits independent of the core count
        return _pod_recipe(sc, seed, M, n_train, keep_snapshots, workers, eps_pca)


def _pod_recipe(sc, seed, M, n_train, keep_snapshots, workers, eps_pca):
    N = sc.N
    n_train = 2 * N if n_train is None else n_train
    fl = initial_flow(sc)
    tau = time_of_flight(sc, fl["p"], fl["faces"], fl["Ff"], fl["link_cells"], fl["Fl"], fl["phiV"])
    T = sc.n_steps * fl["dt0"]
    s_inj = float(np.max(sc.link_s))
    LW, LO = mobility_profiles(sc, tau, T, M=M, s_inj=s_inj)
    mus = training_parameters(M, n_train, seed)
    P = snapshots(sc, LW, LO, mus, p0=fl["p"], workers=workers)
    Phi, kept, S = pod_bases(sc, P, N, eps_pca=eps_pca)
    return OfflineResult(Phi=Phi, kept=kept, sigma=S, tau=tau, T=T, dt0=fl["dt0"], mus=mus, LW=LW, LO=LO,
                         P=P if keep_snapshots else None)
