"""CPU oracle of the LRBMS online step (arXiv 1405.2810) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product path
(``paper_1405_2810_b200``) never imports, links or executes it, and it shares
no code with the CUDA library (only the seeded inputs from
``paper_1405_2810_b200.inputs``, which hold none of the method's arithmetic).

Plain, slow, obviously-correct fp64 NumPy/SciPy.  Every function cites the
PAPER.md passage (``P:line``) it follows and the DESIGN.md reading (R1-R6,
A1-A21) where the paper is silent.  Library primitives used as single steps:
sparse/dense matrix products, dense Cholesky (LAPACK), banded Cholesky
(LAPACK ``pbsv``), sparse LU (SuperLU, fine solves only).

Fine space: k = 0 (one value per cell; reading R1 / A1).  Cells are indexed
c = i + nx (j + ny k) (x fastest); subdomain E = I + Sx (J + Sy L); local cell
l = lx + sx (ly + sy lz).

Pins: every function here is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_pins.py`` (P1-P14 of DESIGN.md); none is "parity unpinned"
except the PCG path's iteration count (its *result* is pinned against the
direct solvers, P13).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

# ----------------------------------------------------------------------------
# a1: mobilities and fractional flow
# ----------------------------------------------------------------------------


def effective_saturation(s, sc):
    """S_e = clamp((s - Swr)/(1 - Swr - Sor), 0, 1)   (reading R5 / A8: clamp only inside k_r)."""
    return np.clip((np.asarray(s, np.float64) - sc.swr) / (1.0 - sc.swr - sc.sor), 0.0, 1.0)


def phase_mobilities(s, sc):
    """lambda_w = k_rw(s)/mu_w, lambda_n = k_ro(s)/mu_n   (eq:brooksCorey).

    k_rw = S_e^nw, k_ro = (1-S_e)^no (Corey; nw = no = 1 is the paper's linear law P:965-966).
    """
    se = effective_saturation(s, sc)
    lam_w = se ** sc.nw / sc.mu_w
    lam_n = (1.0 - se) ** sc.no / sc.mu_o
    return lam_w, lam_n


def total_mobility(s, sc):
    """lambda_t = lambda_w + lambda_n   (eq:brooksCorey)."""
    lam_w, lam_n = phase_mobilities(s, sc)
    return lam_w + lam_n


def fractional_flow(s, sc):
    """f_w = lambda_w / (lambda_w + lambda_n)   (eq:frationalFlow)."""
    lam_w, lam_n = phase_mobilities(s, sc)
    return lam_w / (lam_w + lam_n)


def fractional_flow_derivative(s, sc):
    """d f_w / d s, written out from eq:frationalFlow with the Corey k_r (R5)."""
    se = effective_saturation(s, sc)
    scale = 1.0 / (1.0 - sc.swr - sc.sor)
    a = se ** sc.nw / sc.mu_w
    b = (1.0 - se) ** sc.no / sc.mu_o
    da = sc.nw * se ** (sc.nw - 1.0) / sc.mu_w
    db = -sc.no * (1.0 - se) ** (sc.no - 1.0) / sc.mu_o
    return scale * (da * b - a * db) / (a + b) ** 2


def fprime_max(sc):
    """max_{s in [Swr, 1-Sor]} f_w'(s): the CFL wave-speed bound (reading R4 / A10).

    Dense sampling followed by golden-section refinement of the best bracket.
    """
    lo, hi = sc.swr, 1.0 - sc.sor
    xs = np.linspace(lo, hi, 20001)
    vals = fractional_flow_derivative(xs, sc)
    k = int(np.argmax(vals))
    a, b = xs[max(k - 1, 0)], xs[min(k + 1, len(xs) - 1)]
    g = (np.sqrt(5.0) - 1.0) / 2.0
    for _ in range(200):
        c = b - g * (b - a)
        d = a + g * (b - a)
        if fractional_flow_derivative(c, sc) >= fractional_flow_derivative(d, sc):
            b = d
        else:
            a = c
        if b - a < 1e-15:
            break
    best = max(float(fractional_flow_derivative(0.5 * (a + b), sc)), float(vals[k]))
    return best


# ----------------------------------------------------------------------------
# fine grid topology and coarse partition
# ----------------------------------------------------------------------------


def cell_volume(sc):
    return sc.hx * sc.hy * sc.hz


def face_geometry(sc, axis):
    """|F| / d_F for an interior face normal to ``axis`` (centre-to-centre distance; reading A3)."""
    h = (sc.hx, sc.hy, sc.hz)
    area = h[(axis + 1) % 3] * h[(axis + 2) % 3]
    return area / h[axis]


def interior_faces(sc):
    """Interior faces in global order: x-faces, then y-, then z-faces; within an axis
    ordered by the first cell T1 (normal n_F points from T1 to T2 = T1 + e_axis).

    Returns (a, b, axis) int arrays.
    """
    nx, ny, nz = sc.nx, sc.ny, sc.nz
    idx = np.arange(sc.n).reshape(nz, ny, nx)
    A, B, X = [], [], []
    if nx > 1:
        A.append(idx[:, :, :-1].reshape(-1)); B.append(idx[:, :, 1:].reshape(-1))
        X.append(np.full(A[-1].shape, 0))
    if ny > 1:
        A.append(idx[:, :-1, :].reshape(-1)); B.append(idx[:, 1:, :].reshape(-1))
        X.append(np.full(A[-1].shape, 1))
    if nz > 1:
        A.append(idx[:-1, :, :].reshape(-1)); B.append(idx[1:, :, :].reshape(-1))
        X.append(np.full(A[-1].shape, 2))
    if not A:
        e = np.zeros(0, np.int64)
        return e, e, e
    return np.concatenate(A), np.concatenate(B), np.concatenate(X)


def subdomain_cells(sc):
    """cells[E, l]: global fine cell of local cell l in subdomain E (matching partition).

    E = I + Sx (J + Sy L), l = lx + sx (ly + sy lz), cell = (I sx + lx) + nx ((J sy + ly) + ny (L sz + lz)).
    """
    L, J, I = np.meshgrid(np.arange(sc.Sz), np.arange(sc.Sy), np.arange(sc.Sx), indexing="ij")
    lz, ly, lx = np.meshgrid(np.arange(sc.sz), np.arange(sc.sy), np.arange(sc.sx), indexing="ij")
    I, J, L = I.reshape(-1, 1), J.reshape(-1, 1), L.reshape(-1, 1)
    lx, ly, lz = lx.reshape(1, -1), ly.reshape(1, -1), lz.reshape(1, -1)
    return ((I * sc.sx + lx) + sc.nx * ((J * sc.sy + ly) + sc.ny * (L * sc.sz + lz))).astype(np.int64)


def upper_neighbours(sc):
    """nb[E, d]: subdomain E + e_d (d = 0..dim-1) or -1 at the domain boundary."""
    nb = -np.ones((sc.n_s, sc.dim), np.int64)
    for L in range(sc.Sz):
        for J in range(sc.Sy):
            for I in range(sc.Sx):
                E = I + sc.Sx * (J + sc.Sy * L)
                if I + 1 < sc.Sx:
                    nb[E, 0] = E + 1
                if J + 1 < sc.Sy:
                    nb[E, 1] = E + sc.Sx
                if sc.dim == 3 and L + 1 < sc.Sz:
                    nb[E, 2] = E + sc.Sx * sc.Sy
    return nb


# ----------------------------------------------------------------------------
# a2: fine operator A(lambda), b(lambda)  (SWIP at k = 0 with the lambda-weighted penalty, R2)
# ----------------------------------------------------------------------------


def face_weights(sc, lam):
    """w_F(lambda) = T_F (tau_a lambda_a + tau_b lambda_b)   (reading R2).

    T_F = |F|/d_F * 2 K_a K_b / (K_a + K_b) is the penalty sigma_F/h_F of eq:penaltyParam
    (c_F = 1, a_l = K_l) and tau_l = K_l/(K_a + K_b) the weights of the mean
    {.}.  Affine in lambda (the property the Remark P:312-320 protects).
    """
    a, b, ax = interior_faces(sc)
    K = sc.K
    geo = np.array([face_geometry(sc, d) for d in range(3)])[ax] if len(ax) else np.zeros(0)
    T = geo * 2.0 * K[a] * K[b] / (K[a] + K[b])
    tau_a = K[a] / (K[a] + K[b])
    tau_b = K[b] / (K[a] + K[b])
    return T * (tau_a * lam[a] + tau_b * lam[b])


def link_weights(sc, lam):
    """g_L = (2 |F| / h) K_a lambda_a for a Dirichlet face / well link at cell a (reading R6):
    a SWIP Dirichlet face with tau = 1 at distance h/2."""
    a = sc.link_cell.astype(np.int64)
    geo = np.array([2.0 * face_geometry(sc, d) for d in range(3)])[sc.link_axis]
    return geo * sc.K[a] * lam[a]


def fine_operator(sc, lam):
    """A(lambda) p = b(lambda): the k = 0 pressure system of def:pressureDG.

    A = sum_F w_F (e_a - e_b)(e_a - e_b)^T + sum_L g_L e_a e_a^T,  b = sum_L g_L p_L e_a.
    (Volume and consistency terms of eq:swipBilP vanish for piecewise constants.)
    """
    n = sc.n
    a, b, _ = interior_faces(sc)
    w = face_weights(sc, lam)
    g = link_weights(sc, lam)
    lc = sc.link_cell.astype(np.int64)
    rows = np.concatenate([a, b, a, b, lc])
    cols = np.concatenate([a, b, b, a, lc])
    vals = np.concatenate([w, w, -w, -w, g])
    A = sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr()
    rhs = np.zeros(n)
    np.add.at(rhs, lc, g * sc.link_p)
    return A, rhs


# ----------------------------------------------------------------------------
# a2: Galerkin projection onto the reduced broken space (def:coarseScalePressure)
# ----------------------------------------------------------------------------


def project(sc, A, rhs):
    """B_EE' = Phi_E^T A[E, E'] Phi_E' and r_E = Phi_E^T b[E]   (def:coarseScalePressure P:621-631).

    Returns blocks[E, 0] = B_EE, blocks[E, 1 + d] = B_{E, E + e_d} (0 if no neighbour), r[E].
    Phi is in the ABI layout Phi[E][k][l] (basis function k of E at local cell l).
    """
    cells = subdomain_cells(sc)
    nb = upper_neighbours(sc)
    perm = cells.reshape(-1)
    Ap = A[perm][:, perm].tocsr()
    bp = rhs[perm]
    nl, N = sc.n_loc, sc.N
    blocks = np.zeros((sc.n_s, 1 + sc.dim, N, N))
    r = np.zeros((sc.n_s, N))
    for E in range(sc.n_s):
        PE = sc.Phi[E]
        AEE = Ap[E * nl:(E + 1) * nl, E * nl:(E + 1) * nl].toarray()
        blocks[E, 0] = PE @ AEE @ PE.T
        r[E] = PE @ bp[E * nl:(E + 1) * nl]
        for d in range(sc.dim):
            F = nb[E, d]
            if F >= 0:
                AEF = Ap[E * nl:(E + 1) * nl, F * nl:(F + 1) * nl].toarray()
                blocks[E, 1 + d] = PE @ AEF @ sc.Phi[F].T
    return blocks, r


def reduced_matrix(sc, blocks, dense=False):
    """The reduced matrix B of eq:reducedSystem, assembled from the upper blocks
    (symmetric: B_E'E = B_EE'^T)."""
    nb = upper_neighbours(sc)
    N, R = sc.N, sc.n_s * sc.N
    if dense:
        B = np.zeros((R, R))
        for E in range(sc.n_s):
            B[E * N:(E + 1) * N, E * N:(E + 1) * N] = blocks[E, 0]
            for d in range(sc.dim):
                F = nb[E, d]
                if F >= 0:
                    B[E * N:(E + 1) * N, F * N:(F + 1) * N] = blocks[E, 1 + d]
                    B[F * N:(F + 1) * N, E * N:(E + 1) * N] = blocks[E, 1 + d].T
        return B
    brow, bcol, bdat = [], [], []
    for E in range(sc.n_s):
        brow.append(E); bcol.append(E); bdat.append(blocks[E, 0])
        for d in range(sc.dim):
            F = nb[E, d]
            if F >= 0:
                brow.append(E); bcol.append(F); bdat.append(blocks[E, 1 + d])
                brow.append(F); bcol.append(E); bdat.append(blocks[E, 1 + d].T)
    order = np.lexsort((np.array(bcol), np.array(brow)))
    brow = np.array(brow)[order]; bcol = np.array(bcol)[order]
    bdat = np.stack(bdat)[order]
    indptr = np.searchsorted(brow, np.arange(sc.n_s + 1))
    return sp.bsr_matrix((bdat, bcol, indptr), shape=(R, R)).tocsr()


# ----------------------------------------------------------------------------
# a3: reduced solve  B c = r   (eq:reducedSystem P:818-821; exact-solve reading A17)
# ----------------------------------------------------------------------------


def solve_dense(sc, blocks, r):
    """Dense Cholesky (LAPACK potrf/potrs) of the assembled SPD reduced matrix."""
    B = reduced_matrix(sc, blocks, dense=True)
    cf = sla.cho_factor(B, lower=True, check_finite=True)
    return sla.cho_solve(cf, r.reshape(-1)).reshape(sc.n_s, sc.N)


def solve_banded(sc, blocks, r):
    """Banded Cholesky (LAPACK pbsv) with subdomains ordered x-fastest (bandwidth (Sx+1)N-1)."""
    B = reduced_matrix(sc, blocks, dense=False).tocoo()
    R = sc.n_s * sc.N
    kd = int(np.max(B.row - B.col))
    ab = np.zeros((kd + 1, R))
    low = B.row >= B.col
    ab[B.row[low] - B.col[low], B.col[low]] = B.data[low]
    return sla.solveh_banded(ab, r.reshape(-1), lower=True).reshape(sc.n_s, sc.N)


def solve_pcg(sc, blocks, r, x0=None, rtol=1e-15, maxiter=20000, return_iters=False):
    """Preconditioned conjugate gradients (Hestenes-Stiefel) to stagnation.

    Preconditioner: additive two-level -- exact inverse of each diagonal block B_EE plus a
    coarse correction on the subdomain-indicator coefficients z_E = Phi_E 1_E.
    Only the iteration count depends on it; the converged result is pinned against the
    direct solvers (P13).
    """
    B = reduced_matrix(sc, blocks, dense=False)
    N, ns = sc.N, sc.n_s
    rhs = r.reshape(-1)
    Dinv = np.linalg.inv(blocks[:, 0])
    Z = sc.Phi.sum(axis=2)                      # [E][k]: coefficients of 1_E
    Zs = sp.csr_matrix((Z.reshape(-1), (np.arange(ns * N), np.repeat(np.arange(ns), N))),
                       shape=(ns * N, ns))
    Bc = (Zs.T @ (B @ Zs)).toarray()
    cf = sla.cho_factor(Bc, lower=True)

    def prec(v):
        y = np.einsum("eij,ej->ei", Dinv, v.reshape(ns, N)).reshape(-1)
        return y + Zs @ sla.cho_solve(cf, Zs.T @ v)

    x = np.zeros_like(rhs) if x0 is None else x0.reshape(-1).copy()
    res = rhs - B @ x
    z = prec(res)
    p = z.copy()
    rz = res @ z
    bnorm = np.linalg.norm(rhs)
    it = 0
    for it in range(1, maxiter + 1):
        q = B @ p
        alpha = rz / (p @ q)
        x += alpha * p
        res -= alpha * q
        if np.linalg.norm(res) <= rtol * bnorm:
            break
        z = prec(res)
        rz_new = res @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    out = x.reshape(ns, N)
    return (out, it) if return_iters else out


def solve_reduced(sc, blocks, r, method=None, x0=None):
    R = sc.n_s * sc.N
    if method is None:
        method = "dense" if R <= 4096 else ("banded" if sc.dim == 2 else "pcg")
    if method == "dense":
        return solve_dense(sc, blocks, r)
    if method == "banded":
        return solve_banded(sc, blocks, r)
    if method == "pcg":
        return solve_pcg(sc, blocks, r, x0=x0)
    raise ValueError(method)


# ----------------------------------------------------------------------------
# a4: reconstruction p_h^r = sum_i (p_N)_i phi_i   (alg:fullTwoPhaseScheme step (b))
# ----------------------------------------------------------------------------


def reconstruct(sc, c):
    cells = subdomain_cells(sc)
    p = np.zeros(sc.n)
    for E in range(sc.n_s):
        p[cells[E]] = sc.Phi[E].T @ c[E]
    return p


# ----------------------------------------------------------------------------
# a5: face fluxes (eq:velocityDG P:366-377 at k = 0) and the CFL step (R4)
# ----------------------------------------------------------------------------


def fluxes(sc, p, lam):
    """int_F u.n = w_F (p_a - p_b) on interior faces (n from T1 = a to T2 = b),
    g_L (p_a - p_L) on links (positive = out of the domain): eq:velocityDG at k = 0,
    with the true lambda(s^n) (A9)."""
    a, b, _ = interior_faces(sc)
    Ff = face_weights(sc, lam) * (p[a] - p[b])
    lc = sc.link_cell.astype(np.int64)
    Fl = link_weights(sc, lam) * (p[lc] - sc.link_p)
    return Ff, Fl


def cell_flux_bound(sc, Ff, Fl):
    """Q_i = max(sum of outgoing fluxes, sum of incoming fluxes) of cell i (R4)."""
    a, b, _ = interior_faces(sc)
    lc = sc.link_cell.astype(np.int64)
    out_pos = np.zeros(sc.n)
    out_neg = np.zeros(sc.n)
    # flux leaving cell a is +F, leaving cell b is -F
    np.add.at(out_pos, a, np.maximum(Ff, 0.0)); np.add.at(out_neg, a, np.maximum(-Ff, 0.0))
    np.add.at(out_pos, b, np.maximum(-Ff, 0.0)); np.add.at(out_neg, b, np.maximum(Ff, 0.0))
    np.add.at(out_pos, lc, np.maximum(Fl, 0.0)); np.add.at(out_neg, lc, np.maximum(-Fl, 0.0))
    return np.maximum(out_pos, out_neg)


def cfl_time_step(sc, Ff, Fl, fpmax):
    """dt^n = CFL min_i phi_i V_i / (f'_max Q_i) over cells with Q_i > 0 (reading R4 / A10)."""
    Q = cell_flux_bound(sc, Ff, Fl)
    phi = np.ones(sc.n) if sc.phi is None else sc.phi
    mask = Q > 0
    if not np.any(mask):
        raise FloatingPointError("no flow: max Q = 0")
    return float(sc.cfl * np.min(phi[mask] * cell_volume(sc) / (fpmax * Q[mask])))


# ----------------------------------------------------------------------------
# a6: explicit upwind transport (eq:saturationDG P:389-399 at k = 0, eq:upwind P:400-417)
# ----------------------------------------------------------------------------


def transport(sc, s, Ff, Fl, dt):
    """phi V (s^{n+1} - s^n)/dt = - sum_F F_F f(chi(s^n))  (outward sign per cell).

    Upwind chi: s|T1 if u.n >= 0 else s|T2; on links s_ext on inflow (F < 0),
    the cell value on outflow.  The jump-penalty term of P:397 is dropped (reading A5).
    """
    a, b, _ = interior_faces(sc)
    lc = sc.link_cell.astype(np.int64)
    s_up = np.where(Ff >= 0.0, s[a], s[b])
    flux_w = Ff * fractional_flow(s_up, sc)
    s_up_l = np.where(Fl >= 0.0, s[lc], sc.link_s)
    flux_wl = Fl * fractional_flow(s_up_l, sc)
    net = np.zeros(sc.n)
    np.add.at(net, a, flux_w)
    np.add.at(net, b, -flux_w)
    np.add.at(net, lc, flux_wl)
    phi = np.ones(sc.n) if sc.phi is None else sc.phi
    return s - dt / (phi * cell_volume(sc)) * net


# ----------------------------------------------------------------------------
# the paper's affine online variant (NEXT-1): theta fit + precomputed reduced quantities
# ----------------------------------------------------------------------------


def profile_mobilities(sc, s_profiles):
    """lambda_{t,q} = lambda_{w,q} + lambda_{n,q} of the profile saturation fields (eq:parameterizedMob
    P:570-589, profiles of P:650-662; the total mobility is what eq:leastSquaresFit fits)."""
    return np.stack([total_mobility(sq, sc) for sq in s_profiles])


def theta_fit(sc, lam, lam_q):
    """eq:leastSquaresFit: Theta(s) = argmin_theta || lambda_t(s) - sum_q theta_q
    lambda_{t,q} ||_{l2} over the fine degrees of freedom (k = 0: cells).  Library LAPACK lstsq."""
    theta, *_ = np.linalg.lstsq(np.asarray(lam_q).T, lam, rcond=None)
    return theta


def affine_offline(sc, lam_q):
    """Offline quantities of sec:offlineOnlineDecomposition as reduced blocks:
    b_q = Phi^T A(lambda_{t,q}) Phi, d_q = Phi^T b(lambda_{t,q}).  Under reading R2 the k = 0 operator
    and its Dirichlet right-hand side are linear in lambda (no lambda-free penalty term): c = 0, e = 0."""
    bq, dq = [], []
    for lq in lam_q:
        A, rhs = fine_operator(sc, lq)
        b, r = project(sc, A, rhs)
        bq.append(b)
        dq.append(r)
    return np.stack(bq), np.stack(dq)


def affine_system(theta, bq, dq):
    """eq:reducedSystem with c = e = 0: (sum_q theta_q b_q) p_H = sum_q theta_q d_q."""
    return np.tensordot(theta, bq, axes=1), np.tensordot(theta, dq, axes=1)


# the online step (alg:fullTwoPhaseScheme P:846-882 with direct projection, reading R3)
# ----------------------------------------------------------------------------


def lrbms_step(sc, s, fpmax=None, method=None, x0=None, dt_fixed=0.0, affine=None):
    """One online LRBMS step: (a1) lambda(s^n); (a2) assemble + project; (a3) reduced solve;
    (a4) reconstruct p; (a5) fluxes + dt; (a6) upwind transport.  Returns a dict.
    affine = (lam_q, bq, dq): the paper's variant instead of (a2) (alg:fullTwoPhaseScheme step (a),
    P:863-868): theta fit (eq:leastSquaresFit) and the affine reduced system (eq:reducedSystem); the
    fluxes still use the true lambda(s^n)."""
    if fpmax is None:
        fpmax = fprime_max(sc)
    lam = total_mobility(s, sc)
    theta = None
    if affine is None:
        A, rhs = fine_operator(sc, lam)
        blocks, r = project(sc, A, rhs)
    else:
        lam_q, bq, dq = affine
        theta = theta_fit(sc, lam, lam_q)
        blocks, r = affine_system(theta, bq, dq)
    c = solve_reduced(sc, blocks, r, method=method, x0=x0)
    p = reconstruct(sc, c)
    Ff, Fl = fluxes(sc, p, lam)
    dt = dt_fixed if dt_fixed > 0 else cfl_time_step(sc, Ff, Fl, fpmax)
    s_new = transport(sc, s, Ff, Fl, dt)
    return dict(s=s_new, p=p, c=c, dt=dt, blocks=blocks, r=r, Ff=Ff, Fl=Fl, theta=theta)


def run(sc, n_steps=None, method=None, keep=False, dt_fixed=0.0, s_profiles=None):
    """alg:fullTwoPhaseScheme step 5 for n = 0..n_steps-1 from s^0 = sc.s0 (k = 0 projection of
    s_0 is the cell value).  Returns final state and per-step logs.  s_profiles: the
    profile saturation fields of the paper's affine variant (NEXT-1), else the direct projection."""
    n_steps = sc.n_steps if n_steps is None else n_steps
    fpmax = fprime_max(sc)
    affine = None
    if s_profiles is not None:
        lam_q = profile_mobilities(sc, s_profiles)
        affine = (lam_q,) + affine_offline(sc, lam_q)
    s = np.array(sc.s0, np.float64)
    dts, cs, ps = [], [], []
    out = None
    c_prev = None
    for _ in range(n_steps):
        out = lrbms_step(sc, s, fpmax=fpmax, method=method, x0=c_prev, dt_fixed=dt_fixed, affine=affine)
        s = out["s"]
        c_prev = out["c"]
        dts.append(out["dt"])
        if keep:
            cs.append(out["c"]); ps.append(out["p"])
    res = dict(s=s, dts=np.array(dts), last=out)
    if keep:
        res["cs"] = cs
        res["ps"] = ps
    return res


# ----------------------------------------------------------------------------
# the high-dimensional scheme at k = 0 (alg:highDimTwoPhaseFlow P:471-493, no limiter at k = 0)
# ----------------------------------------------------------------------------


def fine_pressure(sc, s):
    """def:pressureDG: sparse direct solve of A(lambda(s)) p = b(lambda(s))."""
    lam = total_mobility(s, sc)
    A, rhs = fine_operator(sc, lam)
    return spla.spsolve(A.tocsc(), rhs), lam


def fine_step(sc, s, fpmax=None, dt_fixed=0.0):
    if fpmax is None:
        fpmax = fprime_max(sc)
    p, lam = fine_pressure(sc, s)
    Ff, Fl = fluxes(sc, p, lam)
    dt = dt_fixed if dt_fixed > 0 else cfl_time_step(sc, Ff, Fl, fpmax)
    return dict(s=transport(sc, s, Ff, Fl, dt), p=p, dt=dt, Ff=Ff, Fl=Fl)


# ----------------------------------------------------------------------------
# diagnostics of a step (the paper's fine-grid mass-conservation measure)
# ----------------------------------------------------------------------------


def total_mass(sc, s):
    """sum_i phi_i V_i s_i: the water volume (the quantity eq:saturationDG conserves, pin P3)."""
    phi = np.ones(sc.n) if sc.phi is None else sc.phi
    return float(np.sum(phi * cell_volume(sc) * s))


def face_areas(sc):
    h = (sc.hx, sc.hy, sc.hz)
    return np.array([h[(d + 1) % 3] * h[(d + 2) % 3] for d in range(3)])


def cell_net_outflow(sc, Ff, Fl):
    """int_{dT} u.n dS per cell: the outward total flux over the cell's faces and links."""
    a, b, _ = interior_faces(sc)
    net = np.zeros(sc.n)
    np.add.at(net, a, Ff)
    np.add.at(net, b, -Ff)
    np.add.at(net, sc.link_cell.astype(np.int64), Fl)
    return net


def relative_mass_loss(sc, Ff, Fl):
    """zeta(T) = |int_{dT} u.n dS| / max_{x in dT} |u(x)|.  At k = 0 the velocity on a
    face is represented by its normal flux density F_F/|F|, so the max runs over the cell's faces and
    links (reading A33)."""
    a, b, ax = interior_faces(sc)
    area = face_areas(sc)
    umax = np.zeros(sc.n)
    u = np.abs(Ff) / area[ax] if len(ax) else np.zeros(0)
    np.maximum.at(umax, a, u)
    np.maximum.at(umax, b, u)
    lc = sc.link_cell.astype(np.int64)
    np.maximum.at(umax, lc, np.abs(Fl) / area[sc.link_axis])
    net = cell_net_outflow(sc, Ff, Fl)
    return np.where(umax > 0, np.abs(net) / np.where(umax > 0, umax, 1.0), 0.0)


def link_water_outflow(sc, s, Fl):
    """sum_L F_L f(s_up): the water leaving through links in one step (eq:upwind on links)."""
    s_up = np.where(Fl >= 0.0, s[sc.link_cell.astype(np.int64)], sc.link_s)
    return float(np.sum(Fl * fractional_flow(s_up, sc)))
