"""NEXT-4 on the GPU: the LRBMS online step on the k = 1 SWIP-DG fine space (lrbms_k1_*) against the
k = 1 oracle (oracle/k1_oracle.py, pinned in tests/test_k1_pins.py), element by element through the
C ABI: projected blocks and right-hand side (1e-12), then runs with the limiter (dt, c, p1 relative
1e-10, s1 absolute 1e-10, the same cells flagged in the last step)."""
import numpy as np
import pytest

from paper_1405_2810_b200 import inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

K1 = pytest.importorskip("oracle.k1_oracle")
O = pytest.importorskip("oracle.lrbms_oracle")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1405_2810_b200 import build
    build.build()


def np_(t):
    return t.detach().cpu().numpy()


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def case(name):
    if name == "2d":
        return inputs.custom_scenario(12, 8, 1, 4, 4, 1, 6, mu_o=5.0, seed=1, basis1="poly1", cfl=0.2)
    if name == "3d_aniso":   # ragged 3D, anisotropic cells, several chunks with a ragged tail (n_loc = 18)
        return inputs.custom_scenario(6, 6, 4, 3, 3, 2, 8, mu_o=3.0, seed=2, hx=0.5, hy=2.0, hz=1.5,
                                      basis1="poly1", cfl=0.2)
    if name == "wells2d":
        return inputs.custom_scenario(8, 8, 1, 4, 4, 1, 5, mu_o=10.0, seed=4, bc="corner_wells_2d",
                                      basis1="poly1", cfl=0.2)
    if name == "big_sub":    # one subdomain spans several 32-cell chunks (n_loc = 100) and N is not a multiple of 8
        return inputs.custom_scenario(20, 10, 1, 10, 10, 1, 11, mu_o=10.0, seed=5, basis1="poly1", cfl=0.2)
    if name == "single":     # a single subdomain (no couplings, no coarse level)
        return inputs.custom_scenario(6, 5, 1, 6, 5, 1, 7, mu_o=2.0, seed=6, basis1="poly1", cfl=0.2)
    if name == "C1":
        return inputs.make_scenario_k1("C1")
    if name == "C2":
        return inputs.make_scenario_k1("C2")
    raise ValueError(name)


def ctx_k1(sc, s1=None, **solver):
    from paper_1405_2810_b200.lrbms import LrbmsContext
    ctx = LrbmsContext(sc, solver=solver or None, k1_only=True)
    ctx.k1_set_basis(sc.Phi1)
    ctx.k1_set_saturation(K1.initial_saturation(sc) if s1 is None else s1)
    return ctx


def random_p1_saturation(sc, seed):
    rng = np.random.default_rng(seed)
    s1 = np.zeros((sc.dim + 1, sc.n))
    s1[0] = rng.uniform(0.05, 0.95, sc.n)
    s1[1:] = rng.uniform(-0.05, 0.05, (sc.dim, sc.n))
    return s1


@pytest.mark.parametrize("name", ["2d", "3d_aniso", "wells2d", "big_sub", "single", "C1", "C2"])
def test_k1_projection_matches_oracle(name):
    sc = case(name)
    s1 = random_p1_saturation(sc, 11)
    ctx = ctx_k1(sc, s1)
    blocks, r = ctx.k1_stage_project()
    lam = K1.cell_mobility(sc, s1)
    A, b = K1.fine_operator(sc, lam)
    ob, orr = K1.project(sc, A, b)
    assert rel(np_(blocks), ob) <= 1e-12
    assert rel(np_(r), orr) <= 1e-12
    # B_EE exactly symmetric (mirrored tiles)
    d = np_(blocks)[:, 0]
    assert np.array_equal(d, d.transpose(0, 2, 1))


@pytest.mark.parametrize("name,steps", [("2d", 20), ("3d_aniso", 15), ("wells2d", 20), ("big_sub", 20),
                                        ("single", 10), ("C1", 20), ("C2", 30)])
def test_k1_run_matches_oracle(name, steps):
    sc = case(name)
    ref = K1.run(sc, steps, keep=True)
    ctx = ctx_k1(sc, rtol=1e-13)
    dts = np_(ctx.k1_run(steps, log_dt=True))
    s1, p1, c, nflag = ctx.k1_get_state()
    e = dict(dt=rel(dts, ref["dts"]), c=rel(np_(c), ref["cs"][-1]), p=rel(np_(p1), ref["ps"][-1]),
             s=float(np.max(np.abs(np_(s1) - ref["s"]))))
    print(f"k1 {name} {steps} steps: " + ", ".join(f"{k} {v:.3e}" for k, v in e.items()),
          f"flagged {nflag} (oracle {int(ref['last']['flagged'].sum())})")
    assert e["c"] <= 1e-10 and e["p"] <= 1e-10 and e["s"] <= 1e-10 and e["dt"] <= 1e-8
    assert nflag == int(ref["last"]["flagged"].sum())


def test_k1_limiter_acts_and_can_be_switched_off():
    """A sharp front (s = 1 in the first column of cells) flags cells; without the limiter the same
    steps match the oracle's unlimited scheme."""
    sc = case("2d")
    s1 = K1.initial_saturation(sc)
    s1[0, np.arange(sc.n) % sc.nx == 0] = 1.0
    for lim in (True, False):
        ref = K1.run(sc, 8, keep=True, limiter=lim, s1=s1)
        ctx = ctx_k1(sc, s1, rtol=1e-14)
        ctx.k1_run(8, limiter=lim)
        g1, _, _, nflag = ctx.k1_get_state()
        assert float(np.max(np.abs(np_(g1) - ref["s"]))) <= 1e-10
        assert nflag == int(ref["last"]["flagged"].sum())
        if lim:
            assert nflag > 0
        else:
            assert nflag == 0


def test_k1_full_local_basis_is_the_fine_scheme():
    """Phi1_E = the whole local P1 space: the reduced scheme on the GPU equals the oracle's fine
    k = 1 scheme (sparse direct solve), the k = 1 analogue of pin P1."""
    sc = inputs.custom_scenario(6, 4, 1, 2, 2, 1, 1, mu_o=5.0, seed=3, basis1="full1", cfl=0.2)
    sc.N = sc.Phi1.shape[1]
    assert sc.N == 12
    ref = K1.run(sc, 10, fine=True, keep=True)
    ctx = ctx_k1(sc, rtol=1e-14)
    ctx.k1_run(10)
    s1, p1, _, _ = ctx.k1_get_state()
    assert rel(np_(p1), ref["ps"][-1]) <= 1e-10
    assert float(np.max(np.abs(np_(s1) - ref["s"]))) <= 1e-10


def test_k1_deterministic_and_dt_fixed():
    sc = case("wells2d")
    out = []
    for _ in range(2):
        ctx = ctx_k1(sc)
        ctx.k1_run(6, dt_fixed=0.05)
        out.append(np_(ctx.k1_get_state()[0]))
    assert np.array_equal(out[0], out[1])
    ref = K1.run(sc, 6, dt_fixed=0.05)
    assert float(np.max(np.abs(out[0] - ref["s"]))) <= 1e-10


def test_k1_porosity_field():
    """A porosity field enters the CFL step and the mass matrix of the transport (phi |T|)."""
    sc = case("3d_aniso")
    sc.phi = np.random.default_rng(1).uniform(0.1, 0.3, sc.n)
    ref = K1.run(sc, 8, keep=True)
    ctx = ctx_k1(sc, rtol=1e-13)
    dts = np_(ctx.k1_run(8, log_dt=True))
    s1, p1, _, nflag = ctx.k1_get_state()
    assert rel(dts, ref["dts"]) <= 1e-8
    assert rel(np_(p1), ref["ps"][-1]) <= 1e-10
    assert float(np.max(np.abs(np_(s1) - ref["s"]))) <= 1e-10
    assert nflag == int(ref["last"]["flagged"].sum())


def test_k1_errors():
    from paper_1405_2810_b200.lrbms import LrbmsContext, LrbmsError, LRBMS_E_CONFIG, LRBMS_E_STATE
    sc = case("2d")
    ctx = LrbmsContext(sc, k1_only=True)
    with pytest.raises(LrbmsError) as e:
        ctx.k1_run(1)
    assert e.value.status == LRBMS_E_STATE
    ctx.k1_set_basis(sc.Phi1)
    with pytest.raises(LrbmsError) as e:
        ctx.k1_run(1)
    assert e.value.status == LRBMS_E_STATE
    with pytest.raises(LrbmsError) as e:
        ctx.k1_set_basis(sc.Phi1, c_pen=0.0)
    assert e.value.status == LRBMS_E_CONFIG
    # a link on an interior cell is not a Dirichlet face (A29)
    sc2 = case("2d")
    sc2.link_cell = sc2.link_cell.copy()
    sc2.link_cell[0] = 1 + sc2.nx      # an interior cell
    ctx2 = LrbmsContext(sc2, k1_only=True)
    with pytest.raises(LrbmsError) as e:
        ctx2.k1_set_basis(sc2.Phi1)
    assert e.value.status == LRBMS_E_CONFIG


def test_k0_steps_after_k1_need_the_k0_basis_again():
    from paper_1405_2810_b200.lrbms import LrbmsContext, LrbmsError, LRBMS_E_STATE
    sc = case("2d")
    ctx = LrbmsContext(sc)
    ctx.k1_set_basis(sc.Phi1)
    ctx.k1_set_saturation(K1.initial_saturation(sc))
    ctx.k1_run(2)
    with pytest.raises(LrbmsError) as e:
        ctx.run(1)
    assert e.value.status == LRBMS_E_STATE
    ctx.set_basis(sc.Phi)
    ctx.set_saturation(sc.s0)
    ref = O.run(sc, n_steps=5, keep=True)
    ctx.run(5)
    s, _, _ = ctx.get_state()
    assert float(np.max(np.abs(np_(s) - ref["s"]))) <= 1e-10
    # ... and the other way round: the k = 0 basis (and a new medium) invalidate the k = 1 setup
    with pytest.raises(LrbmsError) as e:
        ctx.k1_run(1)
    assert e.value.status == LRBMS_E_STATE
    ctx.k1_set_basis(sc.Phi1)
    ctx.k1_set_saturation(K1.initial_saturation(sc))
    ref1 = K1.run(sc, 3)
    ctx.k1_run(3)
    assert float(np.max(np.abs(np_(ctx.k1_get_state()[0]) - ref1["s"]))) <= 1e-10
