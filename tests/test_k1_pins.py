"""Pins of the k = 1 SWIP-DG oracle (oracle/k1_oracle.py, NEXT-4) against things other than itself:
a brute-force quadrature assembly written from the definitions (basis functions evaluated at Gauss
points, jumps and weighted means formed pointwise), exact reproduction of affine pressures, the
O(h^2) L2 convergence of a manufactured solution, local conservation of the reconstructed
velocity, free-stream preservation, exactness of the transport on linear profiles, the discrete mass
balance, the limiter's mean preservation and a hand-worked limiter case."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import k1_oracle as K1
from oracle import lrbms_oracle as O
from paper_1405_2810_b200 import inputs

G3 = (np.array([-np.sqrt(0.6), 0.0, np.sqrt(0.6)]) / 2.0, np.array([5.0, 8.0, 5.0]) / 18.0)


# ---------------------------------------------------------------------------- brute force
def _basis(sc, c, x):
    """values and gradients of the nd basis functions of cell c at the physical point x."""
    h = (sc.hx, sc.hy, sc.hz)
    i, j, k = c % sc.nx, (c // sc.nx) % sc.ny, c // (sc.nx * sc.ny)
    b = ((i + 0.5) * h[0], (j + 0.5) * h[1], (k + 0.5) * h[2])
    val = [1.0] + [(x[d] - b[d]) / h[d] for d in range(sc.dim)]
    grad = [np.zeros(3)] + [np.eye(3)[d] / h[d] for d in range(sc.dim)]
    return val, grad


def _box_points(lo, hi, dims):
    """tensor 3-point Gauss on the box [lo, hi] over the listed axes (others fixed at lo)."""
    pts = [(np.array(lo, float), 1.0)]
    for d in dims:
        new = []
        for x, w in pts:
            for g, wg in zip(*G3):
                y = x.copy()
                y[d] = 0.5 * (lo[d] + hi[d]) + g * (hi[d] - lo[d])
                new.append((y, w * wg * (hi[d] - lo[d])))
        pts = new
    return pts


def brute_force_system(sc, lam, weights="ern"):
    """a(v, w) and b(w) of eq:swipBilP / P:324-333 by quadrature of the definitions."""
    n, dim, nd = sc.n, sc.dim, sc.dim + 1
    h = (sc.hx, sc.hy, sc.hz)
    A = np.zeros((nd * n, nd * n))
    b = np.zeros(nd * n)
    mu = max(sc.mu_w, sc.mu_o)
    for c in range(n):
        i, j, k = c % sc.nx, (c // sc.nx) % sc.ny, c // (sc.nx * sc.ny)
        lo = np.array([i * h[0], j * h[1], k * h[2]])
        hi = lo + np.array(h)
        for x, w in _box_points(lo, hi if dim == 3 else np.array([hi[0], hi[1], lo[2] + h[2]]), range(dim)):
            w = w * (h[2] if dim == 2 else 1.0)
            _, gr = _basis(sc, c, x)
            for p in range(nd):
                for q in range(nd):
                    A[p * n + c, q * n + c] += w * lam[c] * sc.K[c] * gr[p] @ gr[q]

    def face(c1, c2, ax, lo, hi, pD=None):
        """interior face (c1 -> c2, n = e_ax) or, with c2 None, a Dirichlet face of c1 with the
        outward normal n = +-e_ax given by the sign in pD[1]."""
        tang = [d for d in range(dim) if d != ax]
        diam = np.sqrt(sum(h[d] ** 2 for d in tang))
        pts = _box_points(lo, hi, tang)
        if dim == 2:
            pts = [(x, w * h[2]) for x, w in pts]
        nvec = np.eye(3)[ax]
        if c2 is None:
            sgn = pD[1]
            sig = sc.c_pen / mu * sc.K[c1]
            cells, om, jmp = [c1], [1.0], [1.0]
            nvec = sgn * nvec
        else:
            sig = sc.c_pen / mu * 2 * sc.K[c1] * sc.K[c2] / (sc.K[c1] + sc.K[c2])
            if weights == "ern":
                om = [sc.K[c2] / (sc.K[c1] + sc.K[c2]), sc.K[c1] / (sc.K[c1] + sc.K[c2])]
            else:   # the printed tau_l = a_l / (a_1 + a_2)
                om = [sc.K[c1] / (sc.K[c1] + sc.K[c2]), sc.K[c2] / (sc.K[c1] + sc.K[c2])]
            cells, jmp = [c1, c2], [1.0, -1.0]
        for x, w in pts:
            vals = [_basis(sc, cc, x) for cc in cells]
            for s1, cc1 in enumerate(cells):
                for p in range(nd):
                    jp = jmp[s1] * vals[s1][0][p]
                    mp = om[s1] * lam[cc1] * sc.K[cc1] * (vals[s1][1][p] @ nvec)
                    for s2, cc2 in enumerate(cells):
                        for q in range(nd):
                            jq = jmp[s2] * vals[s2][0][q]
                            mq = om[s2] * lam[cc2] * sc.K[cc2] * (vals[s2][1][q] @ nvec)
                            A[p * n + cc1, q * n + cc2] += w * (sig / diam * jp * jq - mp * jq - mq * jp)
                    if c2 is None:
                        b[p * n + cc1] += w * (sig / diam * jp - mp) * pD[0]

    stride = (1, sc.nx, sc.nx * sc.ny)
    nxyz = (sc.nx, sc.ny, sc.nz)
    for c in range(n):
        ijk = (c % sc.nx, (c // sc.nx) % sc.ny, c // (sc.nx * sc.ny))
        for ax in range(dim):
            if ijk[ax] + 1 < nxyz[ax]:
                lo = np.array([ijk[0] * h[0], ijk[1] * h[1], ijk[2] * h[2]])
                lo[ax] += h[ax]
                hi = lo + np.array(h)
                hi[ax] = lo[ax]
                face(c, c + stride[ax], ax, lo, hi)
    sides = K1.link_sides(sc)
    for L in range(sc.n_links):
        c, ax = int(sc.link_cell[L]), int(sc.link_axis[L])
        ijk = (c % sc.nx, (c // sc.nx) % sc.ny, c // (sc.nx * sc.ny))
        lo = np.array([ijk[0] * h[0], ijk[1] * h[1], ijk[2] * h[2]])
        if sides[L] > 0:
            lo[ax] += h[ax]
        hi = lo + np.array(h)
        hi[ax] = lo[ax]
        face(c, None, ax, lo, hi, pD=(float(sc.link_p[L]), float(sides[L])))
    return A, b


@pytest.mark.parametrize("case", ["2d", "3d", "aniso2d", "wells2d"])
def test_assembly_matches_brute_force_quadrature(case):
    if case == "2d":
        sc = inputs.custom_scenario(4, 3, 1, 2, 3, 1, 3, mu_o=5.0, seed=1)
    elif case == "3d":
        sc = inputs.custom_scenario(3, 2, 2, 3, 2, 2, 3, mu_o=3.0, seed=2)
    elif case == "aniso2d":
        sc = inputs.custom_scenario(3, 4, 1, 3, 2, 1, 3, mu_o=2.0, seed=3, hx=0.5, hy=2.0, hz=3.0)
    else:
        sc = inputs.custom_scenario(4, 4, 1, 2, 2, 1, 3, mu_o=10.0, seed=4, bc="corner_wells_2d")
    sc.c_pen = 7.5
    rng = np.random.default_rng(5)
    lam = rng.uniform(0.1, 2.0, sc.n)
    A, b = K1.fine_operator(sc, lam)
    Ab, bb = brute_force_system(sc, lam)
    assert np.max(np.abs(A.toarray() - Ab)) <= 1e-13 * np.max(np.abs(Ab))
    assert np.max(np.abs(b - bb)) <= 1e-13 * np.max(np.abs(bb))


def test_printed_weights_lose_coercivity_ern_weights_keep_it():
    """Reading A26: with the printed tau_l = a_l / (a_1 + a_2) the consistency term of a face between
    contrasting cells scales with the larger K while the harmonic penalty scales with the smaller one,
    so the form is indefinite; Ern's SWIP weights omega_1 = a_2 / (a_1 + a_2) keep it SPD."""
    K = np.array([1.0, 1e4, 1.0, 1e4])
    sc = inputs.custom_scenario(4, 1, 1, 4, 1, 1, 2, K=K, mu_o=1.0)
    lam = np.ones(sc.n)
    Ae, _ = brute_force_system(sc, lam, "ern")
    At, _ = brute_force_system(sc, lam, "printed")
    assert np.linalg.eigvalsh(Ae).min() > 0
    assert np.linalg.eigvalsh(At).min() < 0
    assert np.max(np.abs(K1.fine_operator(sc, lam)[0].toarray() - Ae)) <= 1e-12 * np.abs(Ae).max()


def test_penalty_examples():
    """eq:penaltyParam with the Remark's c_F / max(mu): S:236-239's examples."""
    sc = inputs.custom_scenario(2, 1, 1, 2, 1, 1, 1, mu_o=1.0)
    sc.c_pen = 1.0
    assert K1.penalty(sc, 1.0, 3.0) == pytest.approx(1.5, rel=1e-15)
    assert K1.penalty(sc, 2.0, 2.0) == pytest.approx(2.0, rel=1e-15)
    sc.mu_w, sc.mu_o = 0.00130581, 0.008
    assert K1.penalty(sc, 1.0, 1.0) == pytest.approx(1.0 / 0.008, rel=1e-15)


# ---------------------------------------------------------------------------- pressure
def test_global_affine_energy():
    """For a global affine v (zero jumps) on a grid without Dirichlet faces a(v, v) = int lambda K |grad v|^2
    (consistency and penalty terms vanish)."""
    sc = inputs.custom_scenario(5, 4, 1, 5, 4, 1, 3, seed=3, hx=0.7, hy=1.3)
    sc.link_cell = sc.link_cell[:0]; sc.link_axis = sc.link_axis[:0]
    sc.link_p = sc.link_p[:0]; sc.link_s = sc.link_s[:0]
    lam = np.random.default_rng(1).uniform(0.5, 1.5, sc.n)
    A, _ = K1.fine_operator(sc, lam)
    bx, by, _ = K1.cell_centres(sc)
    v = np.concatenate([2.0 * bx - 3.0 * by + 1.0, 2.0 * sc.hx * np.ones(sc.n), -3.0 * sc.hy * np.ones(sc.n)])
    expect = np.sum(lam * sc.K * sc.hx * sc.hy * sc.hz * (4.0 + 9.0))
    assert v @ (A @ v) == pytest.approx(expect, rel=1e-13)


@pytest.mark.parametrize("dim", [2, 3])
def test_affine_pressure_reproduced(dim):
    """Homogeneous K, uniform s, left p = 1 / right p = 0: p = 1 - x / L exactly (the P1 space
    contains it and SWIP is consistent), on the fine space and with a reduced basis containing
    the subdomains' linear functions."""
    if dim == 2:
        sc = inputs.custom_scenario(8, 6, 1, 4, 3, 1, 6, K=np.full(48, 3.0), mu_o=5.0, basis1="poly1")
    else:
        sc = inputs.custom_scenario(4, 4, 4, 2, 2, 2, 8, K=np.full(64, 2.0), mu_o=5.0, basis1="poly1")
    s1 = K1.initial_saturation(sc)
    p1, _ = K1.fine_pressure(sc, s1)
    bx = K1.cell_centres(sc)[0]
    L = sc.nx * sc.hx
    assert np.max(np.abs(p1[0] - (1 - bx / L))) <= 1e-12
    assert np.max(np.abs(p1[1] + sc.hx / L)) <= 1e-12
    assert np.max(np.abs(p1[2:])) <= 1e-12
    out = K1.lrbms_step(sc, s1)
    assert np.max(np.abs(out["p"] - p1)) <= 1e-12
    # the reconstructed velocity is the uniform Darcy flux lambda K / L through every x face
    lam = O.total_mobility(0.0, sc)
    a, b, ax = O.interior_faces(sc)
    assert np.max(np.abs(out["Ff"][ax == 0] - lam * sc.K[0] / L)) <= 1e-12
    assert np.max(np.abs(out["Ff"][ax != 0])) <= 1e-12


def _manufactured_error(m):
    sc = inputs.custom_scenario(m, m, 1, m, m, 1, 1, K=np.ones(m * m), mu_o=1.0, bc="all_sides",
                                hx=1.0 / m, hy=1.0 / m)
    sc.c_pen = 10.0
    lam = np.ones(sc.n)
    q = lambda x, y, z: 2 * np.pi ** 2 * np.sin(np.pi * x) * np.sin(np.pi * y)
    A, b = K1.fine_operator(sc, lam, source=q)
    p = spla.spsolve(A.tocsc(), b).reshape(3, sc.n)
    bx, by, _ = K1.cell_centres(sc)
    err = 0.0
    for gx, wx in zip(*G3):
        for gy, wy in zip(*G3):
            x, y = bx + gx * sc.hx, by + gy * sc.hy
            ph = p[0] + p[1] * gx + p[2] * gy
            err += np.sum(wx * wy * sc.hx * sc.hy * (np.sin(np.pi * x) * np.sin(np.pi * y) - ph) ** 2)
    return np.sqrt(err)


def test_manufactured_solution_converges_at_order_two():
    """p = sin(pi x) sin(pi y), -div grad p = 2 pi^2 p, p = 0 on the boundary: the k = 1 SWIP
    solution's L2 error falls as h^2."""
    e = [_manufactured_error(m) for m in (16, 32, 64)]
    rates = [np.log2(e[i] / e[i + 1]) for i in range(2)]
    assert e[-1] < 1.5e-3
    assert min(rates) > 1.85 and rates[1] > rates[0], (e, rates)


def test_velocity_locally_conservative():
    """eq:velocityDG at the fine solution: testing def:pressureDG with psi_0 = 1_T gives sum over the
    faces of T of int u.n = 0 (no sources) -- the conservation property the paper relies on."""
    sc = inputs.custom_scenario(8, 6, 1, 4, 3, 1, 4, mu_o=10.0, seed=2, bc="corner_wells_2d")
    s1 = K1.initial_saturation(sc)
    s1[0] = np.random.default_rng(3).uniform(0, 1, sc.n)
    p1, lam = K1.fine_pressure(sc, s1)
    Ff, Fl = K1.fluxes(sc, p1, lam)
    net = O.cell_net_outflow(sc, Ff, Fl)
    assert np.max(np.abs(net)) <= 1e-12 * np.max(np.abs(Ff))
    assert Fl.sum() == pytest.approx(0.0, abs=1e-12 * np.abs(Fl).max())


# ---------------------------------------------------------------------------- transport
def test_free_stream_preserved():
    """A uniform saturation advected by a conservative velocity stays uniform (mean and slopes),
    when the inflow value equals it."""
    sc = inputs.custom_scenario(8, 6, 1, 4, 3, 1, 4, mu_o=5.0, seed=4, bc="corner_wells_2d")
    sc.link_s[:] = 0.37
    s1 = K1.initial_saturation(sc)
    s1[0] = 0.37
    p1, lam = K1.fine_pressure(sc, s1)
    Ff, Fl = K1.fluxes(sc, p1, lam)
    dt = K1.cfl_time_step(sc, Ff, Fl, O.fprime_max(sc))
    out = K1.transport(sc, s1, Ff, Fl, dt)
    assert np.max(np.abs(out[0] - 0.37)) <= 1e-13   # the cell flux balance is ~1e-15 of the fluxes
    assert np.max(np.abs(out[1:])) <= 1e-13


def test_linear_profile_advected_exactly():
    """Linear f (nw = no = 1, mu_w = mu_o) and a uniform velocity: the P1 upwind DG step is exact on
    s = alpha + beta x (every upwind trace is the continuous value): mean -= dt u beta, slope kept."""
    sc = inputs.custom_scenario(10, 1, 1, 10, 1, 1, 1, mu_o=1.0, nw=1.0, no=1.0)
    alpha, beta, u = 0.2, 0.05, 0.8
    bx = K1.cell_centres(sc)[0]
    s1 = np.stack([alpha + beta * bx, np.full(sc.n, beta * sc.hx), np.zeros(sc.n)])
    sc.link_s[:] = alpha                      # the inflow value at x = 0
    a, b, ax = O.interior_faces(sc)
    Ff = np.full(len(a), u)
    sides = K1.link_sides(sc)
    Fl = sides * u                            # outward: -u at the inlet, +u at the outlet
    dt = 0.3
    out = K1.transport(sc, s1, Ff, Fl, dt)
    assert np.max(np.abs(out[0] - (s1[0] - dt * u * beta))) <= 1e-14
    assert np.max(np.abs(out[1] - s1[1])) <= 1e-14


def test_mass_balance_any_flux_field():
    """sum_T phi |T| (mean^{n+1} - mean^n) = -dt (water through the Dirichlet faces) for arbitrary face
    fluxes and a random P1 saturation: the interior face terms telescope (eq:saturationDG tested with
    psi_0 = 1)."""
    sc = inputs.custom_scenario(6, 5, 1, 3, 5, 1, 3, mu_o=5.0, seed=6)
    rng = np.random.default_rng(7)
    s1 = np.stack([rng.uniform(0, 1, sc.n), rng.uniform(-0.2, 0.2, sc.n), rng.uniform(-0.2, 0.2, sc.n)])
    a, b, ax = O.interior_faces(sc)
    Ff = rng.standard_normal(len(a))
    Fl = rng.standard_normal(sc.n_links)
    dt = 0.01
    out = K1.transport(sc, s1, Ff, Fl, dt)
    sides = K1.link_sides(sc)
    water = 0.0
    for L in range(sc.n_links):   # two-point Gauss on the face; s_D on inflow, the trace on outflow
        c, axL = int(sc.link_cell[L]), int(sc.link_axis[L])
        for g in (-K1.GP, K1.GP):
            tr = s1[0, c] + 0.5 * sides[L] * s1[1 + axL, c] + g * s1[2 - axL, c]
            sv = tr if Fl[L] >= 0 else sc.link_s[L]
            water += 0.5 * Fl[L] * O.fractional_flow(sv, sc)
    V = sc.hx * sc.hy * sc.hz
    assert np.sum(V * (out[0] - s1[0])) == pytest.approx(-dt * water, rel=1e-12, abs=1e-15)


# ---------------------------------------------------------------------------- limiter
def test_limiter_preserves_means_and_bounds_slopes():
    """the limiter changes slopes only, never cell means; slopes only shrink."""
    sc = inputs.custom_scenario(8, 8, 1, 4, 4, 1, 3, mu_o=5.0, seed=8)
    rng = np.random.default_rng(9)
    s1 = np.stack([rng.uniform(0, 1, sc.n), rng.uniform(-0.8, 0.8, sc.n), rng.uniform(-0.8, 0.8, sc.n)])
    a, b, ax = O.interior_faces(sc)
    out, flagged = K1.limit(sc, s1, rng.standard_normal(len(a)), rng.standard_normal(sc.n_links))
    assert flagged.any() and not flagged.all()
    assert np.array_equal(out[0], s1[0])
    assert np.all(np.abs(out[1:]) <= np.abs(s1[1:]))
    assert np.array_equal(out[:, ~flagged], s1[:, ~flagged])


def test_limiter_leaves_smooth_linear_field():
    """A continuous linear field inside [0, 1] has no jumps (detector 0) and no range violation."""
    sc = inputs.custom_scenario(8, 8, 1, 4, 4, 1, 3, mu_o=5.0, seed=8)
    bx, by, _ = K1.cell_centres(sc)
    s1 = np.stack([0.1 + 0.05 * bx + 0.04 * by, np.full(sc.n, 0.05), np.full(sc.n, 0.04)])
    sc.link_s[:] = 0.1                       # the field's value on the inflow side x = 0 varies with y:
    a, b, ax = O.interior_faces(sc)
    Ff = np.where(ax == 0, 1.0, 0.0)
    Fl = np.zeros(sc.n_links)               # no boundary inflow in this check
    out, flagged = K1.limit(sc, s1, Ff, Fl)
    assert not flagged.any()
    assert np.array_equal(out, s1)


def test_limiter_hand_case():
    """Three cells in a row, unit cells (h_T = sqrt 2, d = 2), flow +x at unit flux.  Means (0, 0.5, 0.9),
    slopes (0, 0.6, 0).  Cell 1: upstream jump |0 - (0.5 - 0.3)| = 0.2, S = 0.2 / (0.08 * 2 * 2^(1/4))
    = 1.0511 > 1, flagged; m_right = d/g = 0.4 / 0.6, m_left: g = -0.6, d = -0.5 -> 0.5 / 0.6; min 2/3,
    slope 0.6 -> 0.4.  Cell 0 is flagged by its inflow jump |0 - 1| but its only gradient is 0."""
    sc = inputs.custom_scenario(3, 1, 1, 3, 1, 1, 1, mu_o=1.0)
    s1 = np.array([[0.0, 0.5, 0.9], [0.0, 0.6, 0.0], [0.0, 0.0, 0.0]])
    Ff = np.array([1.0, 1.0])
    Fl = np.array([-1.0, 1.0])
    S = K1.shock_detector(sc, s1, Ff, Fl)
    assert S[1] == pytest.approx(0.2 / (0.16 * 2 ** 0.25), rel=1e-14)
    out, flagged = K1.limit(sc, s1, Ff, Fl)
    assert list(flagged) == [True, True, False]
    assert out[1, 1] == pytest.approx(0.4, rel=1e-14)
    assert np.array_equal(out[0], s1[0]) and out[1, 0] == 0.0 and out[1, 2] == 0.0


# ---------------------------------------------------------------------------- the reduced scheme
@pytest.mark.parametrize("dims", [(6, 4, 1, 2, 2, 1), (4, 4, 2, 2, 2, 1)])
def test_full_local_basis_reproduces_fine_scheme(dims):
    """P1 analogue at k = 1: with Phi_E spanning the whole local P1 space the LRBMS step is the fine
    k = 1 step (pressure, fluxes, dt, limited saturation) for several steps."""
    sc = inputs.custom_scenario(*dims, 1, mu_o=5.0, seed=3, basis1="full1")
    rf = K1.run(sc, 6, fine=True, keep=True)
    rr = K1.run(sc, 6, keep=True)
    assert np.max(np.abs(rr["s"] - rf["s"])) <= 1e-12
    assert np.max(np.abs(rr["dts"] / rf["dts"] - 1)) <= 1e-12
    assert np.max(np.abs(rr["ps"][-1] - rf["ps"][-1])) <= 1e-12


def test_reduced_blocks_symmetric_positive_definite():
    sc = inputs.make_scenario_k1("C1")
    s1 = K1.initial_saturation(sc)
    s1[0] = np.random.default_rng(2).uniform(0, 1, sc.n)
    lam = K1.cell_mobility(sc, s1)
    A, b = K1.fine_operator(sc, lam)
    blocks, r = K1.project(sc, A, b)
    B = O.reduced_matrix(sc, blocks, dense=True)
    assert np.max(np.abs(B - B.T)) <= 1e-13 * np.abs(B).max()
    assert np.linalg.eigvalsh(B).min() > 0
    assert np.linalg.eigvalsh(A.toarray()).min() > 0
