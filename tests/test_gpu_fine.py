"""NEXT-2 on the GPU: the fine-scale reference scheme (alg:highDimTwoPhaseFlow P:471-493 at k = 0,
lrbms_run_fine) against the oracle's fine scheme (oracle.fine_step: sparse direct solve of
def:pressureDG P:337-345, then the same fluxes / CFL step / transport).

Tolerances as for the reduced path (BASELINE.json north_star): p relative 1e-10 (max norm),
s absolute 1e-10, dt relative 1e-10.  At C5 size the oracle's direct solve is replaced by
properties that hold at any size: the GPU pressure's residual in the oracle's own operator, and
the oracle's transport applied to the GPU pressure reproducing the GPU saturation.
"""
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


def ctx_for(sc):
    from paper_1405_2810_b200.lrbms import LrbmsContext
    return LrbmsContext(sc)


def np_(t):
    return t.detach().cpu().numpy()


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-300))


CASES = [
    ("C1", lambda: inputs.make_scenario("C1"), 20),
    ("C2", lambda: inputs.make_scenario("C2"), 10),
    ("ragged2d", lambda: inputs.custom_scenario(15, 12, 1, 5, 4, 1, 7, seed=21, mu_o=5.0), 15),
    ("ragged3d", lambda: inputs.custom_scenario(9, 6, 4, 3, 3, 2, 11, seed=22, mu_o=10.0, bc="corner_columns_3d",
                                                hx=0.5, hy=1.5, hz=2.0), 15),
    ("corey3", lambda: inputs.custom_scenario(12, 12, 1, 4, 4, 1, 5, seed=25, nw=3.0, no=1.5, mu_o=2.0,
                                              swr=0.1, sor=0.05), 15),
]


@pytest.mark.parametrize("name,make,steps", CASES, ids=[c[0] for c in CASES])
def test_fine_run_matches_oracle(name, make, steps):
    sc = make()
    fp = O.fprime_max(sc)
    s = sc.s0.copy()
    dts, p = [], None
    for _ in range(steps):
        out = O.fine_step(sc, s, fpmax=fp)
        s, p = out["s"], out["p"]
        dts.append(out["dt"])
    ctx = ctx_for(sc)
    dt_log, iters = ctx.run_fine(steps, log_dt=True, rtol=1e-14)
    sg, pg, _ = ctx.get_state()
    assert iters > 0
    assert rel(np_(pg), p) <= 1e-10
    assert np.max(np.abs(np_(sg) - s)) <= 1e-10
    assert rel(np_(dt_log), np.array(dts)) <= 1e-10
    ctx.close()


def test_fine_run_dt_fixed_and_porosity():
    sc = inputs.custom_scenario(12, 8, 1, 4, 4, 1, 5, seed=7, mu_o=5.0)
    sc.phi = np.random.default_rng(1).uniform(0.1, 0.3, sc.n)
    fp = O.fprime_max(sc)
    s = sc.s0.copy()
    for _ in range(6):
        s = O.fine_step(sc, s, fpmax=fp, dt_fixed=0.05)["s"]
    ctx = ctx_for(sc)
    dt_log, _ = ctx.run_fine(6, dt_fixed=0.05, log_dt=True, rtol=1e-14)
    sg, _, _ = ctx.get_state()
    assert np.all(np_(dt_log) == 0.05)
    assert np.max(np.abs(np_(sg) - s)) <= 1e-10
    ctx.close()


def test_fine_equals_full_basis_lrbms():
    """P1 across the two GPU paths: the reduced scheme with a full local basis is the fine scheme."""
    sc = inputs.custom_scenario(16, 16, 1, 4, 4, 1, 16, seed=5, mu_o=5.0, basis="full")
    a = ctx_for(sc)
    a.run(10)
    sa, pa, _ = a.get_state()
    b = ctx_for(sc)
    b.run_fine(10, rtol=1e-14)
    sb, pb, _ = b.get_state()
    assert np.max(np.abs(np_(sa) - np_(sb))) <= 1e-10
    assert rel(np_(pb), np_(pa)) <= 1e-10
    a.close()
    b.close()


def test_fine_deterministic_and_warm_start():
    sc = inputs.make_scenario("C2")
    outs = []
    for _ in range(2):
        ctx = ctx_for(sc)
        _, it = ctx.run_fine(5, rtol=1e-13)
        s, p, _ = ctx.get_state()
        outs.append((np_(s), np_(p), it))
        ctx.close()
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]
    # a second call continues from the current pressure: the next step needs fewer iterations than
    # a cold first step
    ctx = ctx_for(sc)
    _, cold = ctx.run_fine(1, rtol=1e-13)
    _, warm = ctx.run_fine(1, rtol=1e-13)
    assert warm < cold
    ctx.close()


def test_fine_c5_properties():
    """C5 (1M cells): one fine step; the GPU pressure solves the oracle's own A p = b to the
    requested accuracy, and the oracle's fluxes + CFL + transport applied to it give the GPU's s."""
    sc = inputs.make_scenario("C5")
    ctx = ctx_for(sc)
    dt_log, iters = ctx.run_fine(1, log_dt=True, rtol=1e-12)
    sg, pg, _ = ctx.get_state()
    pg, sg = np_(pg), np_(sg)
    lam = O.total_mobility(sc.s0, sc)
    A, b = O.fine_operator(sc, lam)
    res = A @ pg - b
    d = A.diagonal()
    # preconditioned residual norm against the preconditioned right-hand side (the stopping rule)
    assert np.sqrt(np.dot(res, res / d)) <= 1e-11 * np.sqrt(np.dot(b, b / d))
    Ff, Fl = O.fluxes(sc, pg, lam)
    dt = O.cfl_time_step(sc, Ff, Fl, O.fprime_max(sc))
    s_ref = O.transport(sc, sc.s0, Ff, Fl, dt)
    assert abs(float(np_(dt_log)[0]) - dt) <= 1e-12 * dt
    assert np.max(np.abs(sg - s_ref)) <= 1e-12
    assert iters > 0
    ctx.close()


def test_fine_errors():
    from paper_1405_2810_b200.lrbms import LrbmsError
    sc = inputs.make_scenario("C1")
    ctx = ctx_for(sc)
    with pytest.raises(LrbmsError):
        ctx.run_fine(1, rtol=0.0)
    with pytest.raises(LrbmsError):
        ctx.run_fine(1, rtol=1e-14, max_iters=2)   # cannot converge in 2 iterations: NUMERICAL
    ctx.close()


def test_reduced_steps_after_fine_steps():
    """The fine run borrows the context's coarse level (E = Z^T A Z and its inverse): reduced steps
    that follow on the same context must still match the oracle (the coarse inverse is rebuilt)."""
    sc = inputs.make_scenario("C2")
    fp = O.fprime_max(sc)
    s = sc.s0.copy()
    for _ in range(3):
        s = O.fine_step(sc, s, fpmax=fp)["s"]
    for _ in range(4):
        s = O.lrbms_step(sc, s, fpmax=fp)["s"]
    ctx = ctx_for(sc)
    ctx.run_fine(3, rtol=1e-14)
    ctx.run(4)
    sg, _, _ = ctx.get_state()
    assert np.max(np.abs(np_(sg) - s)) <= 1e-10
    ctx.close()
