"""Pins of the CPU oracle against what the paper and the mathematics fix (P1-P14).

None of these re-types the oracle's formulas: each compares it with a closed form, a paper
constant, a brute-force independent construction, an invariant, or a special case that
reduces to a textbook result.  CPU only (no GPU marker).
"""
import json
import math
import os

import numpy as np
import pytest
from scipy import stats

from oracle import lrbms_oracle as O
from paper_1405_2810_b200 import inputs

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_constants.json")))


def paper_fluid_scenario(nx=4, ny=4):
    sc = inputs.custom_scenario(nx, ny, 1, 2, 2, 1, 2, nw=1.0, no=1.0,
                                mu_w=GOLDEN["mu_w"]["value"], mu_o=GOLDEN["mu_n"]["value"])
    return sc


# ---------------------------------------------------------------- P11: paper constants

def test_p11_paper_lambda_w_at_1():
    """lambda_w(1) = 765.808 with linear k_rw."""
    sc = paper_fluid_scenario()
    lw, ln = O.phase_mobilities(np.array([1.0, 0.0]), sc)
    assert round(lw[0], GOLDEN["lambda_w_at_1"]["digits"]) == GOLDEN["lambda_w_at_1"]["value"]
    assert lw[1] == GOLDEN["lambda_w_at_0"]["value"]
    assert ln[0] == 0.0 and ln[1] == pytest.approx(1.0 / 0.008)


def test_p11_fractional_flow_half():
    sc = paper_fluid_scenario()
    f = O.fractional_flow(np.array([0.5]), sc)[0]
    assert round(f, 5) == GOLDEN["fractional_flow_at_half"]["value"]


def test_p9_equal_viscosity_linear_constant_total_mobility():
    """mu_w = mu_n and linear k_r => lambda_t = 1/mu for every s."""
    sc = inputs.custom_scenario(4, 4, 1, 2, 2, 1, 2, nw=1.0, no=1.0, mu_w=2.0, mu_o=2.0)
    s = np.linspace(-0.3, 1.4, 41)
    assert np.allclose(O.total_mobility(s, sc), 0.5, rtol=0, atol=1e-15)
    assert np.allclose(O.fractional_flow(np.clip(s, 0, 1), sc), np.clip(s, 0, 1), atol=1e-15)


def test_mobility_clamps_outside_unit_interval():
    sc = inputs.custom_scenario(4, 4, 1, 2, 2, 1, 2, mu_o=5.0)
    lam = O.total_mobility(np.array([-0.5, 0.0, 1.0, 1.7]), sc)
    assert lam[0] == lam[1] == 1.0 / 5.0 and lam[2] == lam[3] == 1.0


def test_fprime_max_against_finite_differences():
    """f'_max equals the max secant slope of f on a fine grid (independent of f's derivative)."""
    for mu_o, ex in [(1.0, 2.0), (5.0, 2.0), (10.0, 2.0), (3.0, 1.0)]:
        sc = inputs.custom_scenario(4, 4, 1, 2, 2, 1, 2, mu_o=mu_o, nw=ex, no=ex)
        xs = np.linspace(0, 1, 400001)
        f = O.fractional_flow(xs, sc)
        slope = np.max(np.diff(f) / np.diff(xs))
        assert O.fprime_max(sc) == pytest.approx(slope, rel=1e-4)
        assert O.fprime_max(sc) >= slope * (1 - 1e-12)


def test_fprime_max_closed_form_equal_viscosity_corey2():
    """mu_w = mu_o, Corey 2: f = s^2/(s^2+(1-s)^2); f'(1/2) = 2 is the maximum."""
    sc = inputs.custom_scenario(4, 4, 1, 2, 2, 1, 2, mu_o=1.0)
    assert O.fprime_max(sc) == pytest.approx(2.0, rel=1e-14)


# ---------------------------------------------------------------- residual saturations (R5)

@pytest.mark.parametrize("swr,sor", [(0.1, 0.2), (0.25, 0.05), (0.0, 0.3)])
def test_effective_saturation_residuals_closed_forms(swr, sor):
    """S_e = (s - Swr)/(1 - Swr - Sor) (R5), pinned by values the Corey law fixes without S_e:
    k_rw(Swr) = 0 and k_ro(1 - Sor) = 0 (the residual saturations are immobile), so
    lambda_t(Swr) = 1/mu_o and lambda_t(1 - Sor) = 1/mu_w; at the mobile midpoint
    s = (Swr + 1 - Sor)/2 the effective saturation is 1/2, so Corey 2 gives
    lambda_t = (1/4)/mu_w + (1/4)/mu_o; at the mobile quarter point it gives (1/16)/mu_w + (9/16)/mu_o.
    (A slip such as dividing by 1 - Swr moves the midpoint value.)"""
    mu_w, mu_o = 0.7, 5.0
    sc = inputs.custom_scenario(4, 4, 1, 2, 2, 1, 2, mu_w=mu_w, mu_o=mu_o, swr=swr, sor=sor)
    mid = 0.5 * (swr + 1.0 - sor)
    quarter = swr + 0.25 * (1.0 - swr - sor)
    s = np.array([swr, 1.0 - sor, mid, quarter, swr - 0.05, 1.0 - sor + 0.05])
    lw, ln = O.phase_mobilities(s, sc)
    assert lw[0] == 0.0 and ln[1] == 0.0
    lam = lw + ln
    assert lam[0] == pytest.approx(1.0 / mu_o, rel=1e-15)
    assert lam[1] == pytest.approx(1.0 / mu_w, rel=1e-15)
    assert lam[2] == pytest.approx(0.25 / mu_w + 0.25 / mu_o, rel=1e-14)
    assert lam[3] == pytest.approx(1.0 / 16.0 / mu_w + 9.0 / 16.0 / mu_o, rel=1e-14)
    # outside the mobile range the law is clamped at its end values (A8)
    assert lam[4] == lam[0] and lam[5] == lam[1]
    f = O.fractional_flow(s, sc)
    assert f[0] == 0.0 and f[1] == 1.0
    assert f[2] == pytest.approx((0.25 / mu_w) / (0.25 / mu_w + 0.25 / mu_o), rel=1e-14)


def _fprime_max_corey2_exact(m_ratio, digits=40):
    """max_S f'(S) for Corey 2 with m = mu_w/mu_o, derived by hand independently of the oracle:
    f = S^2/(S^2 + m(1-S)^2)  =>  f'(S) = 2 m S (1-S) / D^2,  D = S^2 + m (1-S)^2.
    d/dS [S(1-S)/D^2] = 0  <=>  h(S) = (1-2S) D - 2 S (1-S) D' = 0, D' = 2S - 2m(1-S):
    a cubic with a single root in (0, 1) at the maximum of f'; found by bisection in 40-digit
    arithmetic (mpmath), then f' evaluated there in the same precision."""
    import mpmath as mp
    mp.mp.dps = digits
    m = mp.mpf(m_ratio)

    def D(S):
        return S * S + m * (1 - S) ** 2

    def h(S):
        return (1 - 2 * S) * D(S) - 2 * S * (1 - S) * (2 * S - 2 * m * (1 - S))

    lo, hi = mp.mpf("1e-30"), 1 - mp.mpf("1e-30")
    assert h(lo) > 0 > h(hi)
    for _ in range(200):
        mid = (lo + hi) / 2
        if h(mid) > 0:
            lo = mid
        else:
            hi = mid
    S = (lo + hi) / 2
    return float(2 * m * S * (1 - S) / D(S) ** 2)


@pytest.mark.parametrize("mu_o", [1.0, 5.0, 10.0])
def test_fprime_max_corey2_exact_maximiser(mu_o):
    """f'_max for the configs' fluids (Corey 2, mu_o/mu_w = 1, 5, 10) against the exact maximiser of
    f' (root of its derivative's numerator in 40-digit arithmetic): <= 1e-13 relative."""
    sc = inputs.custom_scenario(4, 4, 1, 2, 2, 1, 2, mu_w=1.0, mu_o=mu_o)
    exact = _fprime_max_corey2_exact(1.0 / mu_o)
    assert O.fprime_max(sc) == pytest.approx(exact, rel=1e-13)
    if mu_o == 1.0:
        assert exact == pytest.approx(2.0, rel=1e-15)


@pytest.mark.parametrize("swr,sor", [(0.1, 0.2), (0.2, 0.0)])
def test_fprime_max_residual_scaling(swr, sor):
    """With residual saturations f(s) = F((s - Swr)/(1 - Swr - Sor)), so by the chain rule
    f'_max = F'_max / (1 - Swr - Sor), F'_max the exact Corey-2 maximum above."""
    sc = inputs.custom_scenario(4, 4, 1, 2, 2, 1, 2, mu_w=1.0, mu_o=5.0, swr=swr, sor=sor)
    exact = _fprime_max_corey2_exact(1.0 / 5.0) / (1.0 - swr - sor)
    assert O.fprime_max(sc) == pytest.approx(exact, rel=1e-13)


# ---------------------------------------------------------------- SPEC per-operation examples

def test_face_weight_mean_and_harmonic_penalty():
    """tau-weighted mean of traces (3,1) with a = (1,3) is 1.5; the harmonic
    penalty 2 a1 a2/(a1+a2) with a = (1,3) is 1.5.  w_F = penalty * mean = 2.25."""
    sc = inputs.custom_scenario(2, 1, 1, 1, 1, 1, 1, K=np.array([1.0, 3.0]), basis="random")
    assert O.face_weights(sc, np.array([1.0, 1.0]))[0] == pytest.approx(1.5, rel=1e-15)
    assert O.face_weights(sc, np.array([3.0, 1.0]))[0] == pytest.approx(1.5 * 1.5, rel=1e-15)


def test_face_orientation_and_count():
    """2x1 grid: one interior face with normal from cell 0 to cell 1; face count
    nx(ny+1)+ny(nx+1) minus boundary faces."""
    sc = inputs.custom_scenario(2, 1, 1, 1, 1, 1, 1, basis="random")
    a, b, ax = O.interior_faces(sc)
    assert list(a) == [0] and list(b) == [1] and list(ax) == [0]
    sc = inputs.custom_scenario(6, 4, 3, 2, 2, 3, 2)
    a, b, ax = O.interior_faces(sc)
    assert len(a) == 5 * 4 * 3 + 6 * 3 * 3 + 6 * 4 * 2
    assert np.all(b > a)


# ---------------------------------------------------------------- P8: affinity in lambda

def test_p8_operator_affine_in_lambda():
    sc = inputs.custom_scenario(8, 6, 1, 4, 3, 1, 3, seed=3)
    rng = np.random.default_rng(0)
    l1, l2 = rng.uniform(0.1, 2, sc.n), rng.uniform(0.1, 2, sc.n)
    al, be = 0.37, 1.9
    A1, b1 = O.fine_operator(sc, l1)
    A2, b2 = O.fine_operator(sc, l2)
    A3, b3 = O.fine_operator(sc, al * l1 + be * l2)
    D = (A3 - al * A1 - be * A2).toarray()
    assert np.max(np.abs(D)) <= 1e-14 * np.max(np.abs(A3.toarray()))
    assert np.max(np.abs(b3 - al * b1 - be * b2)) <= 1e-14 * np.max(np.abs(b3))


# ---------------------------------------------------------------- P12: brute force

def brute_force_dense(sc, lam):
    """Dense A, b built cell by cell from the 2d/3d neighbour stencil (independent loops)."""
    n = sc.n
    A = np.zeros((n, n)); b = np.zeros(n)
    h = [sc.hx, sc.hy, sc.hz]
    for k in range(sc.nz):
        for j in range(sc.ny):
            for i in range(sc.nx):
                c = i + sc.nx * (j + sc.ny * k)
                for ax, (di, dj, dk) in enumerate([(1, 0, 0), (0, 1, 0), (0, 0, 1)]):
                    ii, jj, kk = i + di, j + dj, k + dk
                    if ii < sc.nx and jj < sc.ny and kk < sc.nz:
                        d = ii + sc.nx * (jj + sc.ny * kk)
                        area = h[(ax + 1) % 3] * h[(ax + 2) % 3]
                        Ka, Kb = sc.K[c], sc.K[d]
                        harm = 2 * Ka * Kb / (Ka + Kb)
                        mean = (Ka * lam[c] + Kb * lam[d]) / (Ka + Kb)
                        w = area / h[ax] * harm * mean
                        A[c, c] += w; A[d, d] += w; A[c, d] -= w; A[d, c] -= w
    for L in range(sc.n_links):
        c = sc.link_cell[L]; ax = sc.link_axis[L]
        area = h[(ax + 1) % 3] * h[(ax + 2) % 3]
        g = area / (h[ax] / 2) * sc.K[c] * lam[c]
        A[c, c] += g; b[c] += g * sc.link_p[L]
    return A, b


def global_basis(sc):
    """Dense global reduced basis matrix: column (E, k) is phi_k^E extended by zero."""
    P = np.zeros((sc.n, sc.n_s * sc.N))
    for E in range(sc.n_s):
        I = E % sc.Sx; J = (E // sc.Sx) % sc.Sy; L = E // (sc.Sx * sc.Sy)
        l = 0
        for lz in range(sc.sz):
            for ly in range(sc.sy):
                for lx in range(sc.sx):
                    c = (I * sc.sx + lx) + sc.nx * ((J * sc.sy + ly) + sc.ny * (L * sc.sz + lz))
                    P[c, E * sc.N:(E + 1) * sc.N] = sc.Phi[E][:, l]
                    l += 1
    return P


@pytest.mark.parametrize("shape", [(8, 8, 1, 4, 4, 1, 5), (4, 4, 4, 2, 2, 2, 4), (6, 9, 1, 3, 3, 1, 4)])
def test_p12_brute_force_projection_and_solve(shape):
    nx, ny, nz, sx, sy, sz, N = shape
    sc = inputs.custom_scenario(nx, ny, nz, sx, sy, sz, N, seed=11, mu_o=5.0, hx=0.7, hy=1.3,
                                hz=0.9 if nz > 1 else 1.0)
    rng = np.random.default_rng(5)
    s = rng.uniform(0, 1, sc.n)
    lam = O.total_mobility(s, sc)
    Ad, bd = brute_force_dense(sc, lam)
    A, b = O.fine_operator(sc, lam)
    assert np.max(np.abs(A.toarray() - Ad)) <= 1e-13 * np.max(np.abs(Ad))
    assert np.max(np.abs(b - bd)) <= 1e-13 * max(1.0, np.max(np.abs(bd)))
    P = global_basis(sc)
    Bd = P.T @ Ad @ P
    rd = P.T @ bd
    blocks, r = O.project(sc, A, b)
    B = O.reduced_matrix(sc, blocks, dense=True)
    assert np.max(np.abs(B - Bd)) <= 1e-13 * np.max(np.abs(Bd))
    assert np.max(np.abs(r.reshape(-1) - rd)) <= 1e-13 * np.max(np.abs(rd))
    cd = np.linalg.solve(Bd, rd)                      # dense LU, independent of Cholesky
    c = O.solve_reduced(sc, blocks, r, method="dense")
    assert np.max(np.abs(c.reshape(-1) - cd)) <= 1e-12 * np.max(np.abs(cd))
    p = O.reconstruct(sc, c)
    assert np.max(np.abs(p - P @ cd)) <= 1e-12 * np.max(np.abs(p))


# ---------------------------------------------------------------- P5: Galerkin orthogonality, SPD

def test_p5_galerkin_orthogonality_and_spd():
    sc = inputs.custom_scenario(16, 12, 1, 4, 4, 1, 6, seed=2, mu_o=10.0)
    s = np.random.default_rng(1).uniform(0, 1, sc.n)
    lam = O.total_mobility(s, sc)
    A, b = O.fine_operator(sc, lam)
    blocks, r = O.project(sc, A, b)
    for E in range(sc.n_s):
        assert np.allclose(blocks[E, 0], blocks[E, 0].T, rtol=0, atol=1e-14 * np.abs(blocks[E, 0]).max())
    B = O.reduced_matrix(sc, blocks, dense=True)
    assert np.all(np.linalg.eigvalsh(B) > 0)
    c = O.solve_reduced(sc, blocks, r)
    p = O.reconstruct(sc, c)
    res = A @ p - b
    P = global_basis(sc)
    assert np.max(np.abs(P.T @ res)) <= 1e-12 * np.max(np.abs(b))


# ---------------------------------------------------------------- P4: coarse conservation

def test_p4_coarse_conservation_with_indicator_in_basis():
    """Sum_{i in E} (A p - b)_i = 0 whenever 1_E in span Phi_E."""
    sc = inputs.custom_scenario(16, 16, 1, 4, 8, 1, 5, seed=4, mu_o=5.0)
    s = np.random.default_rng(2).uniform(0, 1, sc.n)
    lam = O.total_mobility(s, sc)
    A, b = O.fine_operator(sc, lam)
    blocks, r = O.project(sc, A, b)
    p = O.reconstruct(sc, O.solve_reduced(sc, blocks, r))
    res = A @ p - b
    cells = O.subdomain_cells(sc)
    for E in range(sc.n_s):
        assert abs(res[cells[E]].sum()) <= 1e-13 * np.max(np.abs(b))
    # without the indicator (generic random basis) the defect is O(1) -- the pin is not vacuous
    sc.Phi = inputs.random_basis(sc, 9)
    blocks, r = O.project(sc, A, b)
    p = O.reconstruct(sc, O.solve_reduced(sc, blocks, r))
    res = A @ p - b
    assert max(abs(res[cells[E]].sum()) for E in range(sc.n_s)) > 1e-6


# ---------------------------------------------------------------- P2: homogeneous medium

@pytest.mark.parametrize("basis", ["fine", "poly"])
def test_p2_homogeneous_linear_pressure(basis):
    """Homogeneous K, uniform s, p=1 left / p=0 right: p_i = 1 - x_i / L_x at cell centres."""
    nx, ny = 12, 8
    sc = inputs.custom_scenario(nx, ny, 1, 4, 4, 1, 3, K=np.full(nx * ny, 2.5), hx=0.5, hy=2.0)
    s = np.full(sc.n, 0.3)
    x = (np.arange(nx) + 0.5) * sc.hx
    p_exact = np.tile(1.0 - x / (nx * sc.hx), ny)
    if basis == "fine":
        p, _ = O.fine_pressure(sc, s)
    else:
        out = O.lrbms_step(sc, s)
        p = out["p"]
    assert np.max(np.abs(p - p_exact)) <= 1e-13


def test_p2_homogeneous_3d_wells_symmetry():
    """3D homogeneous with corner well columns: the solution is symmetric under the
    point reflection (i,j) -> (nx-1-i, ny-1-j) combined with p -> 1 - p."""
    sc = inputs.custom_scenario(6, 6, 4, 3, 3, 2, 6, K=np.ones(144), bc="corner_columns_3d", basis="full")
    p, _ = O.fine_pressure(sc, np.zeros(sc.n))
    P = p.reshape(4, 6, 6)
    assert np.max(np.abs(P + P[:, ::-1, ::-1] - 1.0)) <= 1e-13


# ---------------------------------------------------------------- P10: layered 1D series resistance

def test_p10_layered_series_resistances():
    nx = 20
    rng = np.random.default_rng(3)
    Kx = np.exp(rng.standard_normal(nx))
    sc = inputs.custom_scenario(nx, 1, 1, 5, 1, 1, 5, K=Kx, basis="full")
    s = np.full(nx, 0.4)
    lam = O.total_mobility(s, sc)[0]
    # series resistances: half cell at each end (2K lam / h), harmonic faces inside
    Rl = 1.0 / (2 * Kx[0] * lam)
    Rf = np.array([(1 / (2 * Kx[i] * lam) + 1 / (2 * Kx[i + 1] * lam)) for i in range(nx - 1)])
    Rr = 1.0 / (2 * Kx[-1] * lam)
    q = 1.0 / (Rl + Rf.sum() + Rr)
    p_exact = 1.0 - q * (Rl + np.concatenate([[0.0], np.cumsum(Rf)]))
    p, _ = O.fine_pressure(sc, s)
    assert np.max(np.abs(p - p_exact)) <= 1e-13
    out = O.lrbms_step(sc, s)                 # full local bases: the same
    assert np.max(np.abs(out["p"] - p_exact)) <= 1e-12
    assert np.allclose(out["Ff"], q, rtol=1e-12)


# ---------------------------------------------------------------- P9: 1D linear advection

def test_p9_linear_advection_binomial():
    """Linear k_r, mu_w = mu_o, 1D homogeneous: s_i^n = P(Bin(n, nu) >= i+1), nu = CFL."""
    nx, nsteps, nu = 30, 12, 0.5
    sc = inputs.custom_scenario(nx, 1, 1, 10, 1, 1, 10, K=np.ones(nx), nw=1.0, no=1.0,
                                mu_w=1.0, mu_o=1.0, cfl=nu, basis="full")
    assert O.fprime_max(sc) == pytest.approx(1.0, abs=1e-15)
    res = O.run(sc, n_steps=nsteps)
    expect = np.array([stats.binom.sf(i, nsteps, nu) for i in range(nx)])
    assert np.max(np.abs(res["s"] - expect)) <= 1e-12


# ---------------------------------------------------------------- P3: discrete mass balance

def test_p3_mass_balance_any_flux_field():
    sc = inputs.custom_scenario(10, 7, 3, 5, 7, 3, 4, seed=6, mu_o=10.0, bc="corner_columns_3d",
                                hx=0.5, hy=1.0, hz=2.0)
    rng = np.random.default_rng(8)
    s = rng.uniform(0, 1, sc.n)
    a, b, _ = O.interior_faces(sc)
    Ff = rng.standard_normal(len(a))
    Fl = rng.standard_normal(sc.n_links)
    dt = 0.01
    s1 = O.transport(sc, s, Ff, Fl, dt)
    V = sc.hx * sc.hy * sc.hz
    lhs = V * np.sum(s1 - s)
    s_up = np.where(Fl >= 0, s[sc.link_cell], sc.link_s)
    rhs = -dt * np.sum(Fl * O.fractional_flow(s_up, sc))
    assert lhs == pytest.approx(rhs, rel=1e-12, abs=1e-15)


# ---------------------------------------------------------------- P1: full local space = fine solve

@pytest.mark.parametrize("shape", [(8, 8, 1, 4, 4, 1), (6, 4, 4, 3, 2, 2)])
def test_p1_full_basis_reproduces_fine_scheme(shape):
    nx, ny, nz, sx, sy, sz = shape
    bc = "left_right" if nz == 1 else "corner_columns_3d"
    sc = inputs.custom_scenario(nx, ny, nz, sx, sy, sz, 1, seed=7, mu_o=5.0, basis="full", bc=bc)
    fp = O.fprime_max(sc)
    s_r = sc.s0.copy(); s_f = sc.s0.copy()
    for _ in range(15):
        r = O.lrbms_step(sc, s_r, fpmax=fp)
        f = O.fine_step(sc, s_f, fpmax=fp)
        assert np.max(np.abs(r["p"] - f["p"])) <= 1e-12
        assert r["dt"] == pytest.approx(f["dt"], rel=1e-11)
        s_r, s_f = r["s"], f["s"]
    assert np.max(np.abs(s_r - s_f)) <= 1e-12


# ---------------------------------------------------------------- P6: bounds of the fine scheme

def test_p6_fine_scheme_stays_in_bounds():
    sc = inputs.make_scenario("C2", n_steps=40)
    fp = O.fprime_max(sc)
    s = sc.s0.copy()
    for _ in range(40):
        s = O.fine_step(sc, s, fpmax=fp)["s"]
        assert s.min() >= -1e-14 and s.max() <= 1 + 1e-14


# ---------------------------------------------------------------- P13: cross-solver agreement

def test_p13_dense_banded_pcg_agree():
    sc = inputs.make_scenario("C2", n_steps=1)
    s = np.random.default_rng(4).uniform(0, 1, sc.n)
    lam = O.total_mobility(s, sc)
    A, b = O.fine_operator(sc, lam)
    blocks, r = O.project(sc, A, b)
    cd = O.solve_reduced(sc, blocks, r, method="dense")
    cb = O.solve_reduced(sc, blocks, r, method="banded")
    cp = O.solve_reduced(sc, blocks, r, method="pcg")
    scale = np.max(np.abs(cd))
    assert np.max(np.abs(cb - cd)) <= 1e-12 * scale
    assert np.max(np.abs(cp - cd)) <= 1e-11 * scale


def test_p13_pcg_3d_agrees_with_dense():
    sc = inputs.custom_scenario(8, 8, 8, 4, 4, 4, 8, seed=12, mu_o=10.0, bc="corner_columns_3d")
    s = np.random.default_rng(4).uniform(0, 1, sc.n)
    lam = O.total_mobility(s, sc)
    A, b = O.fine_operator(sc, lam)
    blocks, r = O.project(sc, A, b)
    cd = O.solve_reduced(sc, blocks, r, method="dense")
    cp = O.solve_reduced(sc, blocks, r, method="pcg")
    assert np.max(np.abs(cp - cd)) <= 1e-11 * np.max(np.abs(cd))


# ---------------------------------------------------------------- P7: metamorphic scaling

def test_p7_viscosity_scaling_leaves_trajectory_invariant():
    """mu_w, mu_o x4 => lambda / 4, fluxes / 4, dt x 4: same s and p (R4)."""
    sc = inputs.make_scenario("C1", n_steps=5)
    r1 = O.run(sc, keep=True)
    sc.mu_w *= 4; sc.mu_o *= 4
    r2 = O.run(sc, keep=True)
    assert np.max(np.abs(r1["s"] - r2["s"])) <= 1e-13
    assert np.allclose(r2["dts"], 4 * r1["dts"], rtol=1e-13)
    assert np.max(np.abs(r1["ps"][-1] - r2["ps"][-1])) <= 1e-13


def test_p7_permeability_scaling_leaves_trajectory_invariant():
    sc = inputs.make_scenario("C1", n_steps=5)
    r1 = O.run(sc, keep=True)
    sc.K = sc.K * 4
    r2 = O.run(sc, keep=True)
    assert np.max(np.abs(r1["s"] - r2["s"])) <= 1e-13
    assert np.allclose(r2["dts"], r1["dts"] / 4, rtol=1e-13)


# ---------------------------------------------------------------- input recipe sanity

def test_inputs_deterministic_and_shaped():
    a = inputs.make_scenario("C2")
    b = inputs.make_scenario("C2")
    assert a.digest() == b.digest()
    z = np.log(a.K) / 1.5
    assert abs(z.mean()) < 1e-10 and abs(z.std() - 1) < 1e-10
    for name in ["C1", "C2", "C3"]:
        sc = inputs.make_scenario(name)
        assert sc.Phi.shape == (sc.n_s, sc.N, sc.n_loc)
        G = np.einsum("eki,eli->ekl", sc.Phi, sc.Phi)
        assert np.max(np.abs(G - np.eye(sc.N))) < 1e-12
        assert np.allclose(sc.Phi[:, 0, :], 1 / math.sqrt(sc.n_loc), atol=1e-14)


# ---------------------------------------------------------------------------- NEXT-1: the paper's
# affine online variant (eq:leastSquaresFit P:581-586, sec:offlineOnlineDecomposition P:784-833)

def _affine_case():
    sc = inputs.custom_scenario(12, 8, 1, 4, 4, 1, 5, seed=31, mu_o=10.0, n_steps=40)
    sp = inputs.profile_saturations(sc, M=6)   # the paper's recipe: time-of-flight thresholds
    return sc, sp, O.profile_mobilities(sc, sp)


def test_profiles_follow_the_recipe():
    """q = 1 is S0, q = M the injected saturation, the fronts grow monotonically."""
    sc, sp, _ = _affine_case()
    assert np.all(sp[0] == 0.0) and np.all(sp[-1] == 1.0)
    filled = [int((q > 0).sum()) for q in sp]
    assert filled == sorted(filled) and filled[1] > 0 and filled[-2] < sc.n
    assert all(np.all(sp[q] >= sp[q - 1]) for q in range(1, len(sp)))   # the fronts are nested
    # the thresholds are the time of flight's, (q - 1) T / (M - 2) with T = n_steps dt^0 (A31): recomputed
    # here from the recipe's time of flight (pinned in tests/test_offline_recipe.py)
    from offline import recipe as R
    fl = R.initial_flow(sc)
    tau = R.time_of_flight(sc, fl["p"], fl["faces"], fl["Ff"], fl["link_cells"], fl["Fl"], fl["phiV"])
    T = sc.n_steps * fl["dt0"]
    for q in range(2, 6):
        assert np.array_equal(sp[q - 1] > 0, tau <= (q - 1) * T / 4)
    # round 1's geometric proxy is still available
    sd = inputs.profile_saturations(sc, M=6, kind="distance")
    assert np.all(sd[0] == 0.0) and np.all(sd[-1] == 1.0) and not np.array_equal(sd, sp)


def test_theta_fit_recovers_an_exact_combination():
    """eq:leastSquaresFit: lambda = sum theta*_q lambda_q (profiles 2..M, full rank) => theta = theta*."""
    sc, sp, lq = _affine_case()
    sub = lq[1:]
    rng = np.random.default_rng(5)
    th = rng.uniform(0.1, 1.0, sub.shape[0])
    lam = th @ sub
    assert np.allclose(O.theta_fit(sc, lam, sub), th, rtol=1e-10, atol=0)
    # and the residual of a generic lambda is l2-orthogonal to every profile (normal equations)
    lam2 = O.total_mobility(rng.uniform(0, 1, sc.n), sc)
    t2 = O.theta_fit(sc, lam2, lq)
    res = lam2 - t2 @ lq
    assert np.max(np.abs(lq @ res)) <= 1e-10 * np.linalg.norm(lam2) * np.linalg.norm(lq)


def test_affine_decomposition_equals_direct_projection():
    """c = e = 0 under reading R2: sum theta_q b_q, sum theta_q d_q equal the direct projection of the
    operator of sum theta_q lambda_q for any theta (the affine splitting eq:parameterizedMob relies on)."""
    sc, sp, lq = _affine_case()
    bq, dq = O.affine_offline(sc, lq)
    th = np.random.default_rng(6).uniform(-0.5, 1.5, lq.shape[0])
    B, r = O.affine_system(th, bq, dq)
    A, rhs = O.fine_operator(sc, th @ lq)
    Bd, rd = O.project(sc, A, rhs)
    assert np.max(np.abs(B - Bd)) <= 1e-13 * np.max(np.abs(Bd))
    assert np.max(np.abs(r - rd)) <= 1e-13 * np.max(np.abs(rd))


def test_affine_step_equals_direct_step_in_span():
    """S:556 offline-online consistency: when lambda(s) lies in the span of the profiles (here s = a
    profile's saturation field) the affine online step reproduces the direct projection."""
    sc, sp, lq = _affine_case()
    bq, dq = O.affine_offline(sc, lq)
    s = sp[3].copy()
    a = O.lrbms_step(sc, s, method="dense", affine=(lq, bq, dq))
    d = O.lrbms_step(sc, s, method="dense")
    assert np.max(np.abs(a["blocks"] - d["blocks"])) <= 1e-12 * np.max(np.abs(d["blocks"]))
    assert np.max(np.abs(a["c"] - d["c"])) <= 1e-10 * np.max(np.abs(d["c"]))
    assert np.max(np.abs(a["s"] - d["s"])) <= 1e-12


# ---------------------------------------------------------------- K6 diagnostics

def test_relative_mass_loss_zero_for_fine_scheme_and_positive_for_reduced():
    """The fine scheme's fluxes are exactly conservative per cell (zeta = 0 up to round-off: each cell's
    row of A p = b), the reduced scheme's are not -- unless the basis is the full local
    space (P1).  Coarse conservation holds either way (P4: the indicator is in every Phi_E)."""
    sc = inputs.make_scenario("C2", basis="poly")
    s = np.random.default_rng(5).uniform(0, 1, sc.n)
    f = O.fine_step(sc, s)
    z_fine = O.relative_mass_loss(sc, f["Ff"], f["Fl"])
    assert np.max(z_fine) <= 1e-11
    r = O.lrbms_step(sc, s)
    z_red = O.relative_mass_loss(sc, r["Ff"], r["Fl"])
    assert np.max(z_red) > 1e-3
    net = O.cell_net_outflow(sc, r["Ff"], r["Fl"])
    coarse = net[O.subdomain_cells(sc)].sum(axis=1)
    assert np.max(np.abs(coarse)) <= 1e-11 * np.sum(np.abs(r["Fl"]))


def test_relative_mass_loss_closed_form():
    """2 x 1 grid with prescribed fluxes: cell 0 has outflow 3 through the face and inflow 1 through its
    link, so |net| = 2 and max |u| = 3 (unit areas): zeta_0 = 2/3; cell 1: face inflow 3, link outflow
    3 -> zeta_1 = 0."""
    sc = inputs.custom_scenario(2, 1, 1, 1, 1, 1, 1, basis="random")
    Ff = np.array([3.0])
    Fl = np.array([-1.0, 3.0])
    z = O.relative_mass_loss(sc, Ff, Fl)
    assert z[0] == pytest.approx(2.0 / 3.0, rel=1e-15) and z[1] == 0.0


def test_mass_and_link_outflow_balance():
    """P3 restated through the diagnostics: mass^{n+1} - mass^n = -dt sum_L F_L f(s_up)."""
    sc = inputs.make_scenario("C2", basis="poly")
    s = np.random.default_rng(6).uniform(0, 1, sc.n)
    r = O.lrbms_step(sc, s)
    dm = O.total_mass(sc, r["s"]) - O.total_mass(sc, s)
    w = O.link_water_outflow(sc, s, r["Fl"])
    assert abs(dm + r["dt"] * w) <= 1e-14 * O.total_mass(sc, s)
