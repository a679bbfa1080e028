"""GPU parity of the K6 diagnostics (lrbms_diagnostics) against the oracle's diagnostics functions."""
import numpy as np
import pytest

from paper_1405_2810_b200 import inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

O = pytest.importorskip("oracle.lrbms_oracle")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1405_2810_b200 import build
    build.build()


def oracle_last_step(sc, n):
    """s^{n-1} and the n-th step's output of the oracle's run."""
    fp = O.fprime_max(sc)
    s = np.array(sc.s0, np.float64)
    c = None
    for _ in range(n - 1):
        r = O.lrbms_step(sc, s, fpmax=fp, x0=c)
        s, c = r["s"], r["c"]
    return s, O.lrbms_step(sc, s, fpmax=fp, x0=c)


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_diagnostics_match_oracle(name):
    from paper_1405_2810_b200.lrbms import LrbmsContext
    sc = inputs.make_scenario(name)
    n = 6
    s_prev, r = oracle_last_step(sc, n)
    ctx = LrbmsContext(sc)
    ctx.run(n)
    d = ctx.diagnostics()
    m0, m1 = O.total_mass(sc, s_prev), O.total_mass(sc, r["s"])
    z = O.relative_mass_loss(sc, r["Ff"], r["Fl"])
    net = O.cell_net_outflow(sc, r["Ff"], r["Fl"])
    coarse = np.max(np.abs(net[O.subdomain_cells(sc)].sum(axis=1)))
    w = O.link_water_outflow(sc, s_prev, r["Fl"])
    qin, qout = np.sum(np.maximum(-r["Fl"], 0)), np.sum(np.maximum(r["Fl"], 0))
    # the mass moves by dt q per step, dt carries the pressure's error amplified by |p| / |dp|
    assert d["mass_prev"] == pytest.approx(m0, rel=1e-9)
    assert d["mass"] == pytest.approx(m1, rel=1e-9)
    assert abs(d["s_min"] - r["s"].min()) <= 1e-10 and abs(d["s_max"] - r["s"].max()) <= 1e-10
    assert abs(d["zeta_max"] - z.max()) <= 1e-8 and abs(d["zeta_mean"] - z.mean()) <= 1e-8
    assert d["zeta_max"] > 1e-3                          # reduced velocities are not conservative per cell
    assert d["coarse_defect"] <= 1e-10 * qin and coarse <= 1e-10 * qin   # P4: 1_E in span Phi_E
    # link fluxes g (p_a - p_L): the pressure's 1e-10 bar is relative to max|p|, a producer cell's p_a
    # can be 1e-2 of it
    assert d["water_out"] == pytest.approx(w, rel=1e-8)
    assert d["q_in"] == pytest.approx(qin, rel=1e-8) and d["q_out"] == pytest.approx(qout, rel=1e-8)
    assert d["dt"] == pytest.approx(r["dt"], rel=1e-8)
    assert d["mass_balance"] <= 1e-14                    # P3
    ctx.close()


def test_diagnostics_fine_scheme_is_conservative():
    """The fine scheme's velocity is conservative per cell up to its solve's residual (zeta ~ 0)."""
    from paper_1405_2810_b200.lrbms import LrbmsContext
    sc = inputs.make_scenario("C2")
    ctx = LrbmsContext(sc)
    ctx.run_fine(3, rtol=1e-14)
    d = ctx.diagnostics()
    assert d["zeta_max"] <= 1e-8 and d["mass_balance"] <= 1e-14
    ctx.close()


def test_diagnostics_need_a_step():
    from paper_1405_2810_b200.lrbms import LrbmsContext, LrbmsError, LRBMS_E_STATE
    sc = inputs.make_scenario("C1")
    ctx = LrbmsContext(sc)
    with pytest.raises(LrbmsError) as e:
        ctx.diagnostics()
    assert e.value.status == LRBMS_E_STATE
    ctx.close()
