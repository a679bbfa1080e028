"""CPU oracle of the k = 1 SWIP-DG fine space and the LRBMS online step on it
-- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import this module.  The product path never imports, links or executes it; it shares no
code with the CUDA library (the k = 0 oracle's topology helpers are reused: same package).

Plain fp64 NumPy/SciPy, one function per method step in the paper's order:

* pressure: eq:swipBilP with the penalty eq:penaltyParam and the Remark's
  lambda-free c_F / max(mu_w, mu_n); right-hand side P:324-333 (no gravity, no Neumann
  data: all configs); def:pressureDG;
* velocity: the normal fluxes of eq:velocityDG on every face (the RT0 field of P:351-356
  is determined by them);
* saturation: eq:saturationDG with the upwind eq:upwind, explicit Euler;
* limiter: the shock detector, the flagging rule, the gradient scales
   and eq:limiterMain;
* LRBMS: def:coarseScalePressure on the P1 dofs, alg:fullTwoPhaseScheme.

Readings: A4 ("-" sign on the consistency terms), A5 (saturation jump penalty
dropped), A25 (mobility = lambda(cell mean of s), piecewise constant), A26 (SWIP weights
omega_1 = a_2 / (a_1 + a_2): the printed tau_l = a_l / (a_1 + a_2) is not coercive for contrasting K,
pinned), A27 (detector: absolute value of each upstream face's jump integral), A28 (eq:limiterMain's
first term is the cell mean), A29 (links are Dirichlet boundary faces on the side of their cell),
A30 (two-point Gauss quadrature per direction in cells and on faces).

Dofs: per cell T the coefficients of psi_0 = 1, psi_a = xi_a = (x_a - b_{T,a}) / h_a (a = 1..dim),
xi in [-1/2, 1/2]: scaled monomials about the barycentre (mass matrix |T| diag(1, 1/12, ..)).
Global dof index a * n + cell (dof-major); subdomain-local index a * n_loc + l.

Pinned in ``tests/test_k1_pins.py`` against brute-force quadrature assembly, exact reproduction of
affine pressures, the O(h^2) convergence of a manufactured solution, free-stream
preservation, exactness on linear profiles, discrete mass balance and the limiter's mean
preservation.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import lrbms_oracle as O

GP = 0.5 / np.sqrt(3.0)   # two-point Gauss abscissae +-GP on [-1/2, 1/2], weights 1/2 each (A30)


def ndof(sc):
    return sc.dim + 1


def spacing(sc):
    return (sc.hx, sc.hy, sc.hz)


def face_area(sc, ax):
    h = spacing(sc)
    return h[(ax + 1) % 3] * h[(ax + 2) % 3]


def face_diam(sc, ax):
    """h_F = diam(F): the segment length in 2D, the rectangle's diagonal in 3D."""
    h = spacing(sc)
    t = [d for d in range(sc.dim) if d != ax]
    return float(np.sqrt(sum(h[d] ** 2 for d in t)))


def cell_diam(sc):
    h = spacing(sc)
    return float(np.sqrt(sum(h[d] ** 2 for d in range(sc.dim))))


def tangential(sc, ax):
    return [d for d in range(sc.dim) if d != ax]


def mu_max(sc):
    return max(sc.mu_w, sc.mu_o)


def penalty(sc, Ka, Kb):
    """sigma_F = (c_F / max(mu_w, mu_n)) 2 a_1 a_2 / (a_1 + a_2), a_l = K_l (eq:penaltyParam P:305-307
    with the Remark P:316-320); a boundary face uses a_1 = a_2 = K of its cell."""
    return sc.c_pen / mu_max(sc) * 2.0 * Ka * Kb / (Ka + Kb)


def link_sides(sc):
    """Reading A29: link L is the boundary face of its cell on the side of its axis where the cell
    touches the domain boundary (-1: the lower face, +1: the upper face)."""
    nxyz = (sc.nx, sc.ny, sc.nz)
    out = np.zeros(sc.n_links, np.int64)
    for L in range(sc.n_links):
        c = int(sc.link_cell[L])
        ijk = (c % sc.nx, (c // sc.nx) % sc.ny, c // (sc.nx * sc.ny))
        ax = int(sc.link_axis[L])
        if ijk[ax] == 0 and nxyz[ax] > 1:
            out[L] = -1
        elif ijk[ax] == nxyz[ax] - 1 and nxyz[ax] > 1:
            out[L] = 1
        else:
            raise ValueError(f"link {L}: cell {c} is not on a boundary face of axis {ax} (A29)")
    return out


def cell_mobility(sc, s1):
    """Reading A25: lambda_T = lambda_t(mean of s on T) (the P1 dof 0 is the cell mean)."""
    return O.total_mobility(s1[0], sc)


# ----------------------------------------------------------------------------
# pressure: eq:swipBilP, the linear form, def:pressureDG
# ----------------------------------------------------------------------------


def _add_outer(rows, cols, vals, u_idx, u_val, v_idx, v_val, scale):
    for i, a in zip(u_idx, u_val):
        for j, b in zip(v_idx, v_val):
            rows.append(i); cols.append(j); vals.append(scale * a * b)


def fine_operator(sc, lam, source=None):
    """A(lambda) p = b(lambda) of def:pressureDG at k = 1 (closed-form integrals on boxes).

    a(v, w) = sum_T int_T lambda K grad v . grad w
              + sum_F sigma_F / h_F int_F [v][w]
              - sum_F int_F ({lambda K grad v . n}[w] + {lambda K grad w . n}[v])      (A4)
    over interior and Dirichlet faces; b(w) = sum_T int_T q_1 w + sum_{F in Gamma_D} int_F
    (sigma_F / h_F w - lambda K grad w . n) p_D.  lam: per cell (A25).
    source: optional callable q_1(x, y, z) (manufactured-solution pins only).
    """
    n, dim, nd = sc.n, sc.dim, ndof(sc)
    h = spacing(sc)
    V = O.cell_volume(sc)
    K = sc.K
    rows, cols, vals = [], [], []
    # volume: lambda_T K_T |T| / h_a^2 on the slope dofs
    for a in range(1, nd):
        idx = a * n + np.arange(n)
        rows.extend(idx); cols.extend(idx); vals.extend(lam * K * V / h[a - 1] ** 2)
    A_, B_, X_ = O.interior_faces(sc)
    for f in range(len(A_)):
        ca, cb, ax = int(A_[f]), int(B_[f]), int(X_[f])
        area, hF = face_area(sc, ax), face_diam(sc, ax)
        sig = penalty(sc, K[ca], K[cb])
        kap = K[ca] * K[cb] / (K[ca] + K[cb])        # omega_1 K_1 = omega_2 K_2 (A26)
        s_ax = (1 + ax) * n
        # [v] at the face centre: v_a0 + v_a,ax / 2 - v_b0 + v_b,ax / 2
        j0_i = [ca, s_ax + ca, cb, s_ax + cb]
        j0_v = [1.0, 0.5, -1.0, 0.5]
        # {lambda K grad v . n} = kappa (lambda_a v_a,ax + lambda_b v_b,ax) / h_ax
        dn_i = [s_ax + ca, s_ax + cb]
        dn_v = [kap * lam[ca] / h[ax], kap * lam[cb] / h[ax]]
        _add_outer(rows, cols, vals, j0_i, j0_v, j0_i, j0_v, sig / hF * area)
        for t in tangential(sc, ax):
            jt_i = [(1 + t) * n + ca, (1 + t) * n + cb]
            _add_outer(rows, cols, vals, jt_i, [1.0, -1.0], jt_i, [1.0, -1.0], sig / hF * area / 12.0)
        _add_outer(rows, cols, vals, dn_i, dn_v, j0_i, j0_v, -area)
        _add_outer(rows, cols, vals, j0_i, j0_v, dn_i, dn_v, -area)
    rhs = np.zeros(nd * n)
    sides = link_sides(sc)
    for L in range(sc.n_links):
        c, ax, sg = int(sc.link_cell[L]), int(sc.link_axis[L]), float(sides[L])
        area, hF = face_area(sc, ax), face_diam(sc, ax)
        sig = penalty(sc, K[c], K[c])
        s_ax = (1 + ax) * n
        j0_i, j0_v = [c, s_ax + c], [1.0, 0.5 * sg]
        dn_i, dn_v = [s_ax + c], [lam[c] * K[c] * sg / h[ax]]
        _add_outer(rows, cols, vals, j0_i, j0_v, j0_i, j0_v, sig / hF * area)
        for t in tangential(sc, ax):
            jt = (1 + t) * n + c
            _add_outer(rows, cols, vals, [jt], [1.0], [jt], [1.0], sig / hF * area / 12.0)
        _add_outer(rows, cols, vals, dn_i, dn_v, j0_i, j0_v, -area)
        _add_outer(rows, cols, vals, j0_i, j0_v, dn_i, dn_v, -area)
        pD = float(sc.link_p[L])
        for i, v in zip(j0_i, j0_v):
            rhs[i] += area * pD * sig / hF * v
        for i, v in zip(dn_i, dn_v):
            rhs[i] -= area * pD * v
    if source is not None:
        rhs += source_vector(sc, source)
    A = sp.coo_matrix((vals, (rows, cols)), shape=(nd * n, nd * n)).tocsr()
    return A, rhs


def cell_centres(sc):
    c = np.arange(sc.n)
    i, j, k = c % sc.nx, (c // sc.nx) % sc.ny, c // (sc.nx * sc.ny)
    return (i + 0.5) * sc.hx, (j + 0.5) * sc.hy, (k + 0.5) * sc.hz


def source_vector(sc, q):
    """int_T q_1 psi_a by tensor 3-point Gauss (manufactured-solution pins only)."""
    g3 = np.array([-np.sqrt(0.6) / 2, 0.0, np.sqrt(0.6) / 2])
    w3 = np.array([5.0, 8.0, 5.0]) / 18.0
    bx, by, bz = cell_centres(sc)
    V = O.cell_volume(sc)
    nd = ndof(sc)
    out = np.zeros(nd * sc.n)
    zs = [(0.0, 1.0)] if sc.dim == 2 else list(zip(g3, w3))
    for xi, wx in zip(g3, w3):
        for eta, wy in zip(g3, w3):
            for zeta, wz in zs:
                val = q(bx + xi * sc.hx, by + eta * sc.hy, bz + zeta * sc.hz) * wx * wy * wz * V
                out[:sc.n] += val
                out[sc.n:2 * sc.n] += val * xi
                out[2 * sc.n:3 * sc.n] += val * eta
                if sc.dim == 3:
                    out[3 * sc.n:] += val * zeta
    return out


def fine_pressure(sc, s1):
    """def:pressureDG at k = 1: sparse direct solve; returns p1 [nd][n] and lambda."""
    lam = cell_mobility(sc, s1)
    A, b = fine_operator(sc, lam)
    return spla.spsolve(A.tocsc(), b).reshape(ndof(sc), sc.n), lam


# ----------------------------------------------------------------------------
# velocity: eq:velocityDG
# ----------------------------------------------------------------------------


def fluxes(sc, p1, lam):
    """int_F u.n dS = int_F -n.{lambda K grad p} + sigma_F / h_F [p]* dS on every face.
    Interior faces: n from T1 to T2 = T1 + e_ax (O.interior_faces order); links: n outward, [p]* =
    p|_F - p_D.  p1: [nd][n]."""
    h = spacing(sc)
    K = sc.K
    A_, B_, X_ = O.interior_faces(sc)
    Ff = np.zeros(len(A_))
    for f in range(len(A_)):
        ca, cb, ax = int(A_[f]), int(B_[f]), int(X_[f])
        area, hF = face_area(sc, ax), face_diam(sc, ax)
        sig = penalty(sc, K[ca], K[cb])
        kap = K[ca] * K[cb] / (K[ca] + K[cb])
        jump = p1[0, ca] + 0.5 * p1[1 + ax, ca] - p1[0, cb] + 0.5 * p1[1 + ax, cb]
        mean_flux = kap * (lam[ca] * p1[1 + ax, ca] + lam[cb] * p1[1 + ax, cb]) / h[ax]
        Ff[f] = area * (-mean_flux + sig / hF * jump)
    sides = link_sides(sc)
    Fl = np.zeros(sc.n_links)
    for L in range(sc.n_links):
        c, ax, sg = int(sc.link_cell[L]), int(sc.link_axis[L]), float(sides[L])
        area, hF = face_area(sc, ax), face_diam(sc, ax)
        sig = penalty(sc, K[c], K[c])
        trace = p1[0, c] + 0.5 * sg * p1[1 + ax, c]
        Fl[L] = area * (-lam[c] * K[c] * sg * p1[1 + ax, c] / h[ax] + sig / hF * (trace - sc.link_p[L]))
    return Ff, Fl


def cfl_time_step(sc, Ff, Fl, fpmax):
    """Reading R4 with the k = 1 face fluxes: CFL min_T phi_T |T| / (f'_max Q_T)."""
    return O.cfl_time_step(sc, Ff, Fl, fpmax)


# ----------------------------------------------------------------------------
# saturation: eq:saturationDG with eq:upwind
# ----------------------------------------------------------------------------


def _face_points(sc, ax):
    """Tangential Gauss points (dicts axis -> xi) and weights (sum 1) on a face normal to ax (A30)."""
    t = tangential(sc, ax)
    pts = [{}]
    for d in t:
        pts = [{**p, d: x} for p in pts for x in (-GP, GP)]
    return pts, 1.0 / len(pts)


def _trace(sc, s1, c, ax, side, pt):
    """Value of the P1 function of cell c on its face (axis ax, side +-1) at tangential point pt."""
    v = s1[0, c] + 0.5 * side * s1[1 + ax, c]
    for d, x in pt.items():
        v += s1[1 + d, c] * x
    return v


def transport(sc, s1, Ff, Fl, dt):
    """One explicit Euler step of eq:saturationDG at k = 1 (A5: no jump penalty):
    int_T phi/dt (s^{n+1} - s^n) v = int_T u f(s^n) . grad v - sum_F int_F (u.n) f(chi(s^n)) [v].
    u is the RT0 field of the face fluxes (u_a linear in xi_a); quadrature A30.  Returns s1 new."""
    n, dim, nd = sc.n, sc.dim, ndof(sc)
    h = spacing(sc)
    V = O.cell_volume(sc)
    phi = np.ones(n) if sc.phi is None else sc.phi
    A_, B_, X_ = O.interior_faces(sc)
    sides = link_sides(sc)
    # flux through each cell's lower / upper face of axis a, in the +e_a direction
    Flo = np.zeros((3, n))
    Fhi = np.zeros((3, n))
    for f in range(len(A_)):
        Fhi[X_[f], A_[f]] = Ff[f]
        Flo[X_[f], B_[f]] = Ff[f]
    for L in range(sc.n_links):
        c, ax = int(sc.link_cell[L]), int(sc.link_axis[L])
        if sides[L] > 0:
            Fhi[ax, c] = Fl[L]
        else:
            Flo[ax, c] = -Fl[L]
    R = np.zeros((nd, n))
    # volume term: int_T u f(s) . grad psi_a = (1/h_a) int_T u_a f(s) dx, tensor 2-point Gauss
    pts = [{}]
    for d in range(dim):
        pts = [{**p, d: x} for p in pts for x in (-GP, GP)]
    w = V / len(pts)
    for pt in pts:
        sv = s1[0].copy()
        for d, x in pt.items():
            sv = sv + s1[1 + d] * x
        fv = O.fractional_flow(sv, sc)
        for a in range(dim):
            ua = (Flo[a] * (0.5 - pt[a]) + Fhi[a] * (0.5 + pt[a])) / face_area(sc, a)
            R[1 + a] += w * ua * fv / h[a]
    # interior faces: - int_F (F/|F|) f(s_up) [v]; [v] = v|T1 for T1, -v|T2 for T2
    for f in range(len(A_)):
        ca, cb, ax = int(A_[f]), int(B_[f]), int(X_[f])
        F = Ff[f]
        pts_f, wf = _face_points(sc, ax)
        for pt in pts_f:
            s_up = _trace(sc, s1, ca, ax, +1, pt) if F >= 0.0 else _trace(sc, s1, cb, ax, -1, pt)
            g = F * wf * O.fractional_flow(s_up, sc)     # (F/|F|) * |F| * weight
            R[0, ca] -= g
            R[0, cb] += g
            R[1 + ax, ca] -= g * 0.5
            R[1 + ax, cb] += g * (-0.5)
            for d, x in pt.items():
                R[1 + d, ca] -= g * x
                R[1 + d, cb] += g * x
    # Dirichlet faces: n outward; chi = s_D on inflow (F < 0), the cell's trace on outflow
    for L in range(sc.n_links):
        c, ax, sg = int(sc.link_cell[L]), int(sc.link_axis[L]), int(sides[L])
        F = Fl[L]
        pts_f, wf = _face_points(sc, ax)
        for pt in pts_f:
            s_up = _trace(sc, s1, c, ax, sg, pt) if F >= 0.0 else sc.link_s[L]
            g = F * wf * O.fractional_flow(s_up, sc)
            R[0, c] -= g
            R[1 + ax, c] -= g * 0.5 * sg
            for d, x in pt.items():
                R[1 + d, c] -= g * x
    mass = np.array([1.0] + [1.0 / 12.0] * dim)
    return s1 + dt * R / (phi * V)[None, :] / mass[:, None]


# ----------------------------------------------------------------------------
# limiter
# ----------------------------------------------------------------------------


def shock_detector(sc, s1, Ff, Fl):
    """S(T) = sum over the upstream faces of T (u.n_T < 0) of |int_F [s] dS| / (0.08 d sqrt(h_T) |T|)
    (A27).  [s] is taken at the face centre (exact: it is linear along F); on a Dirichlet
    inflow face [s]* = s|_T - s_D."""
    n, dim = sc.n, sc.dim
    V = O.cell_volume(sc)
    scale = 1.0 / (0.08 * dim * np.sqrt(cell_diam(sc)) * V)
    S = np.zeros(n)
    A_, B_, X_ = O.interior_faces(sc)
    for f in range(len(A_)):
        ca, cb, ax = int(A_[f]), int(B_[f]), int(X_[f])
        jump = abs((s1[0, ca] + 0.5 * s1[1 + ax, ca]) - (s1[0, cb] - 0.5 * s1[1 + ax, cb]))
        val = face_area(sc, ax) * jump * scale
        if Ff[f] > 0.0:      # flows from a into b: upstream face of b
            S[cb] += val
        elif Ff[f] < 0.0:
            S[ca] += val
    sides = link_sides(sc)
    for L in range(sc.n_links):
        if Fl[L] < 0.0:      # inflow through the Dirichlet face
            c, ax, sg = int(sc.link_cell[L]), int(sc.link_axis[L]), float(sides[L])
            jump = abs(s1[0, c] + 0.5 * sg * s1[1 + ax, c] - sc.link_s[L])
            S[c] += face_area(sc, ax) * jump * scale
    return S


def gradient_scale(g, d):
    """m_i of P:449-456."""
    big = abs(g) > 1e-8 and abs(d) > 1e-8
    if g * d < 0.0 and big:
        return 0.0
    if g * d > 0.0 and abs(g) > abs(d) and big:
        return d / g
    return 1.0


def limit(sc, s1, Ff, Fl):
    """The stabilised saturation of eq:limiterMain (A28): in flagged cells (S(T) > 1 or
    s(x) outside [0, 1] on T) s~ = mean + min_i m_i grad s . (x - b_T), with g_i =
    grad s . (b_i - b_T) = +-(slope dof of the axis) and d_i the difference of the cell means over the
    face neighbours T_i; unflagged cells keep s.  Returns (s1 limited, flagged mask)."""
    n, dim = sc.n, sc.dim
    S = shock_detector(sc, s1, Ff, Fl)
    spread = 0.5 * np.sum(np.abs(s1[1:]), axis=0)
    flagged = (S > 1.0) | (s1[0] - spread < 0.0) | (s1[0] + spread > 1.0)
    out = s1.copy()
    nxyz = (sc.nx, sc.ny, sc.nz)
    stride = (1, sc.nx, sc.nx * sc.ny)
    for c in np.nonzero(flagged)[0]:
        ijk = (c % sc.nx, (c // sc.nx) % sc.ny, c // (sc.nx * sc.ny))
        m = 1.0
        for ax in range(dim):
            for sg in (-1, 1):
                q = ijk[ax] + sg
                if 0 <= q < nxyz[ax]:
                    nb = c + sg * stride[ax]
                    g = sg * s1[1 + ax, c]
                    d = s1[0, nb] - s1[0, c]
                    m = min(m, gradient_scale(g, d))
        out[1:, c] = m * s1[1:, c]
    return out, flagged


# ----------------------------------------------------------------------------
# the schemes
# ----------------------------------------------------------------------------


def fine_step(sc, s1, fpmax=None, dt_fixed=0.0, limiter=True):
    """alg:highDimTwoPhaseFlow step 2 at k = 1: (a) pressure, (b) velocity, (c) saturation,
    (d) limiter."""
    if fpmax is None:
        fpmax = O.fprime_max(sc)
    p1, lam = fine_pressure(sc, s1)
    Ff, Fl = fluxes(sc, p1, lam)
    dt = dt_fixed if dt_fixed > 0 else cfl_time_step(sc, Ff, Fl, fpmax)
    sb = transport(sc, s1, Ff, Fl, dt)
    s_new, flagged = limit(sc, sb, Ff, Fl) if limiter else (sb, np.zeros(sc.n, bool))
    return dict(s=s_new, s_bar=sb, p=p1, dt=dt, Ff=Ff, Fl=Fl, flagged=flagged)


def subdomain_dofs(sc):
    """dofs[E, l']: global dof of local dof l' = a n_loc + l of subdomain E."""
    cells = O.subdomain_cells(sc)
    return np.concatenate([a * sc.n + cells for a in range(ndof(sc))], axis=1)


def project(sc, A, rhs):
    """B_EE' = Phi_E A[E, E'] Phi_E'^T, r_E = Phi_E b[E] on the P1 dofs (def:coarseScalePressure
    P:621-631); sc.Phi1[E] is N x (nd n_loc) in the local dof order a n_loc + l."""
    dofs = subdomain_dofs(sc)
    nb = O.upper_neighbours(sc)
    N = sc.Phi1.shape[1]
    blocks = np.zeros((sc.n_s, 1 + sc.dim, N, N))
    r = np.zeros((sc.n_s, N))
    Acsr = A.tocsr()
    for E in range(sc.n_s):
        PE = sc.Phi1[E]
        AEE = Acsr[dofs[E]][:, dofs[E]].toarray()
        blocks[E, 0] = PE @ AEE @ PE.T
        r[E] = PE @ rhs[dofs[E]]
        for d in range(sc.dim):
            F = nb[E, d]
            if F >= 0:
                blocks[E, 1 + d] = PE @ Acsr[dofs[E]][:, dofs[F]].toarray() @ sc.Phi1[F].T
    return blocks, r


def reconstruct(sc, c):
    """p = sum_E Phi_E^T c_E on the P1 dofs; returns [nd][n]."""
    dofs = subdomain_dofs(sc)
    p = np.zeros(ndof(sc) * sc.n)
    for E in range(sc.n_s):
        p[dofs[E]] = sc.Phi1[E].T @ c[E]
    return p.reshape(ndof(sc), sc.n)


def solve_reduced(sc, blocks, r):
    """Exact reduced solve (A17): dense Cholesky of the assembled SPD matrix (the k = 1 cases are
    small), via the k = 0 oracle's assembly of the block matrix."""
    class _S:
        pass
    t = _S()
    t.n_s, t.N, t.dim = sc.n_s, blocks.shape[2], sc.dim
    t.Sx, t.Sy, t.Sz = sc.Sx, sc.Sy, sc.Sz
    return O.solve_dense(t, blocks, r) if t.n_s * t.N <= 6000 else O.solve_banded(t, blocks, r)


def lrbms_step(sc, s1, fpmax=None, dt_fixed=0.0, limiter=True):
    """The online LRBMS step on the k = 1 fine space: lambda(s^n) (A25), assemble + project, reduced
    solve, reconstruct, velocity, CFL step, transport, limiter (alg:fullTwoPhaseScheme P:863-880 with
    the velocity/saturation/limiter steps of alg:highDimTwoPhaseFlow P:484-491)."""
    if fpmax is None:
        fpmax = O.fprime_max(sc)
    lam = cell_mobility(sc, s1)
    A, b = fine_operator(sc, lam)
    blocks, r = project(sc, A, b)
    c = solve_reduced(sc, blocks, r)
    p1 = reconstruct(sc, c)
    Ff, Fl = fluxes(sc, p1, lam)
    dt = dt_fixed if dt_fixed > 0 else cfl_time_step(sc, Ff, Fl, fpmax)
    sb = transport(sc, s1, Ff, Fl, dt)
    s_new, flagged = limit(sc, sb, Ff, Fl) if limiter else (sb, np.zeros(sc.n, bool))
    return dict(s=s_new, s_bar=sb, p=p1, c=c, dt=dt, Ff=Ff, Fl=Fl, blocks=blocks, r=r, flagged=flagged)


def initial_saturation(sc):
    """alg:highDimTwoPhaseFlow step 1: the L2 projection of a cellwise-constant s_0 onto
    V_h is its cell value with zero slopes."""
    s1 = np.zeros((ndof(sc), sc.n))
    s1[0] = sc.s0
    return s1


def run(sc, n_steps, fine=False, keep=False, dt_fixed=0.0, limiter=True, s1=None):
    fpmax = O.fprime_max(sc)
    s1 = initial_saturation(sc) if s1 is None else np.array(s1, np.float64)
    dts, cs, ps, ss = [], [], [], []
    out = None
    for _ in range(n_steps):
        out = (fine_step if fine else lrbms_step)(sc, s1, fpmax=fpmax, dt_fixed=dt_fixed, limiter=limiter)
        s1 = out["s"]
        dts.append(out["dt"])
        if keep:
            ps.append(out["p"]); ss.append(s1)
            if not fine:
                cs.append(out["c"])
    res = dict(s=s1, dts=np.array(dts), last=out)
    if keep:
        res.update(cs=cs, ps=ps, ss=ss)
    return res
