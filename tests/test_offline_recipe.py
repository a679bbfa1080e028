"""Pins of the host offline basis recipe (offline/recipe.py, basis = "pod"): each step against a
closed form, an independent construction (the oracle's fine operator, a monolithic sparse solve) or
an invariant.  CPU only."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from offline import recipe as R
from oracle import lrbms_oracle as O
from paper_1405_2810_b200 import inputs


def homogeneous(nx, ny, sx, sy, N=2, K=1.0, phi=None, hx=1.0, hy=1.0):
    sc = inputs.custom_scenario(nx, ny, 1, sx, sy, 1, N, K=np.full(nx * ny, K), hx=hx, hy=hy, mu_o=5.0)
    if phi is not None:
        sc.phi = np.full(sc.n, phi)
    return sc


def tof_of(sc):
    fl = R.initial_flow(sc)
    return fl, R.time_of_flight(sc, fl["p"], fl["faces"], fl["Ff"], fl["link_cells"], fl["Fl"], fl["phiV"])


# ---------------------------------------------------------------- time of flight (eq:timeOfFlight P:505-512)

@pytest.mark.parametrize("phi,hx", [(1.0, 1.0), (0.3, 0.5)])
def test_tof_uniform_flow_closed_form(phi, hx):
    """Homogeneous medium, left/right Dirichlet: uniform flux u per face, and the DG0 upwind
    time of flight is tau_i = phi V (i + 1) / u -- phi x/u at the cell's downstream face
    x = (i + 1) h (streamline integral int phi/|v| dx of P:498-501 with v = u/|F|)."""
    sc = homogeneous(12, 6, 4, 3, hx=hx, phi=phi)
    fl, tau = tof_of(sc)
    a, b = fl["faces"]
    ax = (b - a) == 1
    u = fl["Ff"][ax]
    assert np.max(np.abs(u - u[0])) <= 1e-12 * u[0]          # uniform flow
    assert np.max(np.abs(fl["Ff"][~ax])) <= 1e-12 * u[0]      # no transverse flow
    i = np.arange(sc.n) % sc.nx
    V = hx * sc.hy
    exact = phi * V * (i + 1) / u[0]
    assert np.max(np.abs(tau - exact) / exact) <= 1e-12


def test_tof_scaling():
    """tau is linear in phi and inversely proportional to the velocity (K x 2 doubles every flux)."""
    sc = inputs.make_scenario("C2", basis="poly")
    _, t1 = tof_of(sc)
    sc2 = inputs.make_scenario("C2", basis="poly")
    sc2.K = sc2.K * 2.0
    _, t2 = tof_of(sc2)
    sc3 = inputs.make_scenario("C2", basis="poly")
    sc3.phi = np.full(sc3.n, 0.25)
    _, t3 = tof_of(sc3)
    assert np.max(np.abs(t2 * 2.0 - t1) / t1) <= 1e-10
    assert np.max(np.abs(t3 * 4.0 - t1) / t1) <= 1e-10


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_tof_sweep_equals_monolithic_solve(name):
    """The descending-pressure sweep solves the same discrete system as one sparse direct
    solve, and the order is a topological order: every inflow neighbour has a higher p."""
    sc = inputs.make_scenario(name, basis="poly")
    fl, tau = tof_of(sc)
    M, rhs = R.tof_matrix(sc, fl["faces"], fl["Ff"], fl["link_cells"], fl["Fl"], fl["phiV"])
    d = M.diagonal()
    live = d > 0
    Ml = M[live][:, live].tocsc()
    # inflow from stagnant cells is zero (a stagnant cell has no outflow), so the live block is closed
    t_direct = spla.spsolve(Ml, rhs[live])
    assert np.max(np.abs(t_direct - tau[live]) / t_direct) <= 1e-9
    assert np.all(tau[~live] == np.max(tau[live]))
    a, b = fl["faces"]
    F = fl["Ff"]
    up = np.where(F > 0, a, b)
    dn = np.where(F > 0, b, a)
    nz = F != 0
    assert np.all(fl["p"][up[nz]] > fl["p"][dn[nz]])


# ---------------------------------------------------------------- profiles

def test_profiles_structure():
    sc = inputs.make_scenario("C2", basis="poly")
    fl, tau = tof_of(sc)
    T = sc.n_steps * fl["dt0"]
    M = 8
    LW, LO = R.mobility_profiles(sc, tau, T, M=M)
    lw0, lo0 = 0.0, 1.0 / sc.mu_o          # lambda(S0 = 0): only oil moves
    lw1, lo1 = 1.0 / sc.mu_w, 0.0          # lambda(S_inj = 1): only water
    assert np.all(LW[0] == lw0) and np.all(LO[0] == lo0)
    assert np.all(LW[M - 1] == lw1) and np.all(LO[M - 1] == lo1)
    prev = np.zeros(sc.n, bool)
    for q in range(2, M):
        inj = LW[q - 1] == lw1
        assert np.array_equal(inj, tau <= (q - 1) * T / (M - 2))
        assert np.all(LO[q - 1][inj] == lo1) and np.all(LO[q - 1][~inj] == lo0)
        assert np.all(inj[prev])            # the injected region grows with q
        prev = inj
    assert 0 < prev.sum() < sc.n


# ---------------------------------------------------------------- training set

def test_training_parameters():
    mu = R.training_parameters(8, 100_000, 7)
    assert mu.shape == (100_000, 8)
    assert np.max(np.abs(mu.sum(axis=1) - 1.0)) <= 1e-12
    assert mu.min() >= 1e-4 / (1.0 + 8e-4)
    assert np.max(np.abs(mu.mean(axis=0) - 1.0 / 8)) <= 0.01      # uniform on the simplex
    assert np.array_equal(R.training_parameters(8, 20, 105), R.training_parameters(8, 20, 105))
    assert not np.array_equal(R.training_parameters(8, 20, 105), R.training_parameters(8, 20, 106))


# ---------------------------------------------------------------- snapshots and POD

@pytest.mark.parametrize("name", ["C2", "C3"])
def test_snapshots_solve_the_oracle_operator(name):
    """Every snapshot solves the fine system assembled independently by the oracle."""
    sc = inputs.make_scenario(name, basis="poly")
    res = R.pod_recipe(sc, 100 + inputs.CONFIG_INDEX[name], keep_snapshots=True)
    lam = res.mus @ (res.LW + res.LO)
    for j in range(len(res.mus)):
        A, b = O.fine_operator(sc, lam[j])
        r = b - A @ res.P[j]
        assert np.linalg.norm(r) <= 1e-12 * np.linalg.norm(b)


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_pod_basis_orthonormal_with_indicator(name):
    sc = inputs.make_scenario(name, basis="poly")
    res = R.pod_recipe(sc, 100 + inputs.CONFIG_INDEX[name])
    Phi = res.Phi
    assert Phi.shape == (sc.n_s, sc.N, sc.n_loc)
    G = np.einsum("ekl,ejl->ekj", Phi, Phi)
    assert np.max(np.abs(G - np.eye(sc.N)[None])) <= 1e-13
    assert np.max(np.abs(Phi[:, 0, :] - 1.0 / np.sqrt(sc.n_loc))) == 0.0
    assert np.all(res.kept >= 1)


def test_pod_rank_one_when_profiles_coincide():
    """C1 has mu_w = mu_o: the total mobility of every profile is 1, all snapshots coincide, so
    exactly one POD mode survives, proportional to the snapshot with its mean removed."""
    sc = inputs.make_scenario("C1", basis="poly")
    res = R.pod_recipe(sc, 101, keep_snapshots=True)
    assert np.all(res.kept == 1)
    cells = R.local_cells(sc)
    for E in range(sc.n_s):
        y = res.P[0][cells[E]]
        y = y - y.mean()
        u = res.Phi[E, 1]
        assert abs(abs(u @ y) - np.linalg.norm(y)) <= 1e-12 * np.linalg.norm(y)


def test_pod_spans_snapshots_and_reproduces_them():
    """With fewer training parameters than N - 1 nothing is truncated: every snapshot restriction lies
    in span Phi_E (eps_pca = 0: every nonzero mode is kept), so the reduced (oracle) solve at a
    training mobility reproduces that snapshot -- Galerkin reproduction (SPEC 'Reproduction')."""
    sc = inputs.make_scenario("C2", basis="poly")
    res = R.pod_recipe(sc, 102, n_train=5, keep_snapshots=True, eps_pca=0.0)
    cells = R.local_cells(sc)
    for j in range(5):
        for E in range(sc.n_s):
            y = res.P[j][cells[E]]
            Q = res.Phi[E].T
            assert np.linalg.norm(y - Q @ (Q.T @ y)) <= 1e-10 * np.linalg.norm(y)
    sc.Phi = res.Phi
    lam = res.mus @ (res.LW + res.LO)
    for j in (0, 3):
        A, b = O.fine_operator(sc, lam[j])
        blocks, r = O.project(sc, A, b)
        c = O.solve_reduced(sc, blocks, r, method="dense")
        p = O.reconstruct(sc, c)
        assert np.max(np.abs(p - res.P[j])) <= 1e-10 * np.max(np.abs(res.P[j]))


# ---------------------------------------------------------------------------- greedy extension
def _greedy_setup(name="C2", n_train=None):
    sc = inputs.make_scenario(name, basis="poly")
    g = R.greedy_recipe(sc, 100 + inputs.CONFIG_INDEX[name], n_train=n_train)
    return sc, g


def test_greedy_first_round_errors_match_an_independent_reduced_solve():
    """Round 0 of alg:lrbmsBasisConstruction: in the space of the coarse unit functions the
    energy-norm errors of every training mobility, recomputed with the ORACLE's operator,
    projection, reduced solve and reconstruction (N = 1), and the worst approximated parameter."""
    sc, g = _greedy_setup()
    sc1 = inputs.make_scenario("C2", basis="poly")
    sc1.N = 1
    sc1.Phi = np.full((sc1.n_s, 1, sc1.n_loc), 1.0 / np.sqrt(sc1.n_loc))
    A_bar, _ = O.fine_operator(sc1, g["lam_bar"])
    errs = []
    for j in range(len(g["mus"])):
        A, b = O.fine_operator(sc1, g["LAM"][j])
        blocks, r = O.project(sc1, A, b)
        c = O.solve_reduced(sc1, blocks, r, method="dense")
        e = O.reconstruct(sc1, c) - g["P"][j]
        errs.append(np.sqrt(e @ (A_bar @ e)))
    errs = np.array(errs)
    assert g["history"][0][1] == int(np.argmax(errs))
    assert g["history"][0][0] == pytest.approx(errs.max(), rel=1e-9)
    assert g["selected"][0] == int(np.argmax(errs))


def test_greedy_reproduces_selected_snapshots_and_reduces_the_error():
    sc, g = _greedy_setup()
    e0 = g["history"][0][0]
    assert all(g["errors"][j] <= 1e-8 * e0 for j in g["selected"])      # Galerkin: a snapshot in W is reproduced
    assert g["history"][-1][0] <= 1e-2 * e0                              # the training error fell by > 100x
    assert len(set(g["selected"])) == len(g["selected"])
    # the bases: orthonormal, coarse unit function first, sizes between 1 and N
    Phi = g["Phi"]
    G = np.einsum("ekl,ejl->ekj", Phi, Phi)
    assert np.max(np.abs(G - np.eye(sc.N)[None])) <= 1e-12
    assert np.max(np.abs(Phi[:, 0, :] - 1.0 / np.sqrt(sc.n_loc))) <= 1e-15
    assert g["sizes"].min() >= 1 and g["sizes"].max() == sc.N


def test_greedy_with_few_snapshots_spans_what_the_pod_spans():
    """With fewer independent snapshots than N - 1 the greedy uses them all, and its local spaces
    span(v0, snapshots|_E) are the POD's (same projectors on the columns that come from snapshots)."""
    sc, g = _greedy_setup(n_train=4)
    assert sorted(g["selected"]) == [0, 1, 2, 3]
    Phi_p, kept, _ = R.pod_bases(sc, g["P"], sc.N, eps_pca=1e-12)
    for E in range(sc.n_s):
        m = int(g["sizes"][E])
        if m != kept[E] + 1:
            continue            # a restriction at the noise floor: the two rank decisions may differ
        Pg = g["Phi"][E, :m].T @ g["Phi"][E, :m]
        Pp = Phi_p[E, :m].T @ Phi_p[E, :m]
        assert np.max(np.abs(Pg - Pp)) <= 1e-6
    assert np.mean(g["sizes"] == kept + 1) >= 0.9


def test_greedy_stops_at_the_tolerance():
    sc = inputs.make_scenario("C2", basis="poly")
    g = R.greedy_recipe(sc, 102, eps_tol=1e9)
    assert g["selected"] == [] and np.all(g["sizes"] == 1)             # nothing to add: indicators + completion
    G = np.einsum("ekl,ejl->ekj", g["Phi"], g["Phi"])
    assert np.max(np.abs(G - np.eye(sc.N)[None])) <= 1e-12
