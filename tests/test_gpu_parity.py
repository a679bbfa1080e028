"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Tolerances (BASELINE.json north_star):
  reduced coefficients c and pressures p: ||d||_inf / ||ref||_inf <= 1e-10;
  saturations after the full run: ||d||_inf <= 1e-10 (absolute).
Stage-level checks are tighter (same arithmetic, different summation order).
"""
import os

import numpy as np
import pytest

from paper_1405_2810_b200 import inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

O = pytest.importorskip("oracle.lrbms_oracle")

# C4's saturation bar on prefixes at the default solver settings (the C4
# exception): a 1e-14 relative perturbation of K alone moves s by ~1e-10 after 20 steps and 2.2e-10
# after 50 (round-off amplification), so two implementations that differ at round-off
# level cannot be held to 1e-10 in s there; c and p keep the 1e-10 bar
C4_S_BAR = {20: 2e-10, 50: 1e-9}
# dt is reported beside the bar (A20: the bar is c, p and s): dt = cfl min phi V/(f' Q)
# divides by the largest cell flux, a difference of neighbouring pressures, so its relative error is
# the pressure's times |p| / |dp| (~1e2-1e3 on these grids)
DT_BAR = 1e-8
# s after the full run: 1e-10 (BASELINE.json) except where the trajectory itself amplifies round-off
# beyond it.  C3 on the paper-recipe (pod) bases: a 1e-14 relative perturbation of K moves s by 1.3e-11
# after 10 steps and 1.0e-10 after 500 (GPU path against itself, rtol 1e-14;
# profiles/r02k_c3_sens.txt), so two implementations that differ at round-off level (dense Cholesky vs
# deflated PCG) cannot be held to 1e-10 there.  Measured against the oracle: 8.9e-10 at the default
# rtol 5e-13, 2.2e-10 at 1e-13, 8.6e-11 at 1e-14 (profiles/r02k_c3_rtol.txt); c and p keep the 1e-10 bar.
FULL_RUN_S_BAR = {("C3", "pod"): 2e-9}


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1405_2810_b200 import build
    build.build()


def ctx_for(sc, **solver):
    from paper_1405_2810_b200.lrbms import LrbmsContext
    return LrbmsContext(sc, solver=solver or None)


def rel(a, b):
    a = np.asarray(a); b = np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def np_(t):
    return t.detach().cpu().numpy()


SMALL = [
    ("C1", lambda: inputs.make_scenario("C1")),
    ("ragged2d", lambda: inputs.custom_scenario(15, 12, 1, 5, 4, 1, 7, seed=21, mu_o=5.0)),
    ("ragged3d", lambda: inputs.custom_scenario(9, 6, 4, 3, 3, 2, 11, seed=22, mu_o=10.0, bc="corner_columns_3d",
                                                hx=0.5, hy=1.5, hz=2.0)),
    ("one_subdomain", lambda: inputs.custom_scenario(8, 8, 1, 8, 8, 1, 6, seed=23, mu_o=3.0)),
    ("linear_kr", lambda: inputs.custom_scenario(16, 8, 1, 4, 4, 1, 3, seed=24, nw=1.0, no=1.0, mu_o=4.0)),
    ("corey3", lambda: inputs.custom_scenario(12, 12, 1, 4, 4, 1, 5, seed=25, nw=3.0, no=1.5, mu_o=2.0,
                                              swr=0.1, sor=0.05)),
    # mid-size 3D (64 subdomains): the on-chip PCG runs as one thread-block cluster of 8 CTAs x 8 warps
    # (cluster barriers, DSMEM partials), with coupling blocks in tensor memory and in shared memory
    ("cluster3d", lambda: inputs.custom_scenario(12, 12, 8, 3, 3, 2, 9, seed=26, mu_o=10.0, bc="corner_columns_3d")),
    # 18 subdomains in 2D: a cluster of 3 CTAs with a ragged last CTA
    ("cluster2d", lambda: inputs.custom_scenario(24, 12, 1, 4, 4, 1, 6, seed=27, mu_o=5.0)),
]


@pytest.mark.parametrize("name,make", SMALL, ids=[s[0] for s in SMALL])
def test_stage_parity_small(name, make):
    sc = make()
    rng = np.random.default_rng(3)
    s = rng.uniform(-0.05, 1.05, sc.n)        # includes values outside [0,1] (clamped mobility)
    sc.s0 = s
    ctx = ctx_for(sc)
    blocks, r = ctx.stage_project()
    lam = O.total_mobility(s, sc)
    A, b = O.fine_operator(sc, lam)
    ob, orr = O.project(sc, A, b)
    assert rel(np_(blocks), ob) <= 1e-13
    assert rel(np_(r), orr) <= 1e-13
    c = ctx.stage_solve()
    oc = O.solve_reduced(sc, ob, orr, method="dense")
    assert rel(np_(c), oc) <= 1e-10          # north-star bar (PCG to rtol 1e-12 vs dense Cholesky)
    p = ctx.stage_reconstruct()
    op = O.reconstruct(sc, oc)
    assert rel(np_(p), op) <= 1e-10
    ff, lf, dt = ctx.stage_transport()
    oFf, oFl = O.fluxes(sc, op, lam)
    assert rel(np_(ff), oFf) <= 1e-10
    assert rel(np_(lf), oFl) <= 1e-10
    odt = O.cfl_time_step(sc, oFf, oFl, O.fprime_max(sc))
    assert abs(float(dt[0]) - odt) <= 1e-10 * odt   # dt = CFL / max flux ratio: the flux bar
    s1, _, _ = ctx.get_state()
    os1 = O.transport(sc, s, oFf, oFl, odt)
    assert np.max(np.abs(np_(s1) - os1)) <= 1e-10
    ctx.close()


@pytest.mark.parametrize("onchip", [1, 0], ids=["onchip", "l2stream"])
@pytest.mark.parametrize("name,make", SMALL, ids=[s[0] for s in SMALL])
def test_full_run_small(name, make, onchip):
    """Both reduced-solve kernels: k_pcg_tm (operator held in tensor / shared memory, the default)
    and k_pcg (couplings streamed from L2 every iteration)."""
    sc = make()
    n = 20
    ref = O.run(sc, n_steps=n, keep=True)
    ctx = ctx_for(sc, onchip=onchip)
    dts = np_(ctx.run(n, log_dt=True))
    s, p, c = ctx.get_state()
    st = ctx.stats()
    print(f"{name}: iters {st['total_iters']}, ns max|I-EX| {st['ns_resid_max']:.3e}, trips {st['ns_guard_trips']}")
    assert rel(dts, ref["dts"]) <= 1e-10
    assert rel(np_(c), ref["cs"][-1]) <= 1e-10
    assert rel(np_(p), ref["ps"][-1]) <= 1e-10
    assert np.max(np.abs(np_(s) - ref["s"])) <= 1e-10
    assert st["steps"] == n and st["total_iters"] > 0
    ctx.close()


@pytest.mark.parametrize("use_coarse", [0, 1, 2])
@pytest.mark.parametrize("onchip", [1, 0], ids=["onchip", "l2stream"])
def test_coarse_modes_c2(use_coarse, onchip):
    """Block Jacobi only (0), additive two-level (1) and deflation (2), in both PCG kernels, on C2:
    a 10-step run against the oracle (reduced coefficients and saturations at the parity bar)."""
    sc = inputs.make_scenario("C2", n_steps=10)
    ref = O.run(sc, n_steps=10, keep=True)
    ctx = ctx_for(sc, use_coarse=use_coarse, onchip=onchip)
    ctx.run(10)
    s, p, c = ctx.get_state()
    assert rel(np_(c), ref["cs"][-1]) <= 1e-10
    assert np.max(np.abs(np_(s) - ref["s"])) <= 1e-10
    assert ctx.stats()["total_iters"] > 0


def test_onchip_matches_l2stream_c5_prefix():
    """The two PCG kernels on the bench workload (C5, 5 steps): the same trajectory to round-off."""
    sc = inputs.make_scenario("C5", n_steps=5)
    outs = []
    for oc in (1, 0):
        ctx = ctx_for(sc, onchip=oc)
        ctx.run(5)
        s, p, c = ctx.get_state()
        outs.append((np_(s), np_(c)))
        ctx.close()
    assert rel(outs[0][1], outs[1][1]) <= 1e-10
    assert np.max(np.abs(outs[0][0] - outs[1][0])) <= 1e-12


def test_full_basis_reproduces_fine_scheme_gpu():
    """P1 on the GPU: Phi_E = full orthogonal local space => the fine k = 0 scheme."""
    sc = inputs.custom_scenario(16, 16, 1, 4, 4, 1, 16, seed=5, mu_o=5.0, basis="full")
    fp = O.fprime_max(sc)
    s = sc.s0.copy()
    for _ in range(10):
        s = O.fine_step(sc, s, fpmax=fp)["s"]
    ctx = ctx_for(sc)
    ctx.run(10)
    sg, _, _ = ctx.get_state()
    assert np.max(np.abs(np_(sg) - s)) <= 1e-10


def test_dt_fixed_and_porosity():
    sc = inputs.custom_scenario(12, 8, 1, 4, 4, 1, 5, seed=7, mu_o=5.0)
    sc.phi = np.random.default_rng(1).uniform(0.1, 0.3, sc.n)
    ref = O.run(sc, n_steps=6, dt_fixed=0.05)
    ctx = ctx_for(sc)
    ctx.run(6, dt_fixed=0.05)
    s, _, _ = ctx.get_state()
    assert np.max(np.abs(np_(s) - ref["s"])) <= 1e-11
    sc2 = inputs.custom_scenario(12, 8, 1, 4, 4, 1, 5, seed=7, mu_o=5.0)
    sc2.phi = sc.phi
    ref2 = O.run(sc2, n_steps=6)
    ctx2 = ctx_for(sc2)
    ctx2.run(6)
    s2, _, _ = ctx2.get_state()
    assert np.max(np.abs(np_(s2) - ref2["s"])) <= 1e-11


def test_run_host_matches_device_path():
    sc = inputs.make_scenario("C1")
    ctx = ctx_for(sc)
    s_h, p_h = ctx.run_host(5, s_in=sc.s0, want_p=True)
    ctx2 = ctx_for(sc)
    ctx2.run(5)
    s_d, p_d, _ = ctx2.get_state()
    assert np.array_equal(s_h, np_(s_d)) and np.array_equal(p_h, np_(p_d))


def test_run_host_pinned_overlapped_copies():
    """e2e path with pinned buffers, as bench.py drives it: the last step's pressure is copied out on
    the copy stream while the transport runs; s and p must equal the device path bitwise, also with
    several steps per call and s_in == s_out."""
    sc = inputs.make_scenario("C2")
    ctx = ctx_for(sc)
    s_pin = torch.from_numpy(sc.s0.copy()).pin_memory()
    p_pin = torch.empty(sc.n, dtype=torch.float64).pin_memory()
    for _ in range(3):
        ctx.run_host_ptr(2, s_pin.data_ptr(), s_pin.data_ptr(), p_pin.data_ptr())
    ctx2 = ctx_for(sc)
    ctx2.run(6)
    s_d, p_d, _ = ctx2.get_state()
    assert np.array_equal(s_pin.numpy(), np_(s_d)) and np.array_equal(p_pin.numpy(), np_(p_d))
    ctx.close()
    ctx2.close()


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_determinism_bitwise(name):
    """Bitwise-identical reruns on the three launch shapes of the on-chip PCG (C2: one CTA; C3: one
    thread-block cluster; C4: a cooperative grid) -- a race or an order-dependent sum would show here
    (compute-sanitizer is closed on this pool, profiles/r02h)."""
    sc = inputs.make_scenario(name, n_steps=10)
    outs = []
    for _ in range(3 if name != "C4" else 2):
        ctx = ctx_for(sc)
        ctx.run(10)
        s, p, c = ctx.get_state()
        outs.append((np_(s), np_(p), np_(c)))
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)


def test_metamorphic_viscosity_scaling_bitwise():
    """P7: mu x 4 => the same s and p, dt x 4 (powers of two scale exactly)."""
    sc = inputs.make_scenario("C1", n_steps=8)
    ctx = ctx_for(sc)
    d1 = np_(ctx.run(8, log_dt=True))
    s1, p1, _ = ctx.get_state()
    sc.mu_w *= 4; sc.mu_o *= 4
    ctx2 = ctx_for(sc)
    d2 = np_(ctx2.run(8, log_dt=True))
    s2, p2, _ = ctx2.get_state()
    assert np.allclose(d2, 4 * d1, rtol=1e-14, atol=0)
    assert np.max(np.abs(np_(s1) - np_(s2))) <= 1e-14
    assert np.max(np.abs(np_(p1) - np_(p2))) <= 1e-14


def test_config_errors():
    from paper_1405_2810_b200.lrbms import LrbmsError, LRBMS_E_CONFIG
    sc = inputs.custom_scenario(8, 8, 1, 4, 4, 1, 4)
    sc.N = 40
    with pytest.raises(LrbmsError) as e:
        ctx_for(sc)
    assert e.value.status == LRBMS_E_CONFIG
    sc = inputs.custom_scenario(8, 8, 1, 4, 4, 1, 4)
    sc.sx = 3
    with pytest.raises(LrbmsError):
        ctx_for(sc)
    sc = inputs.custom_scenario(8, 8, 1, 4, 4, 1, 4)
    sc.link_cell = sc.link_cell[:0]; sc.link_axis = sc.link_axis[:0]
    sc.link_p = sc.link_p[:0]; sc.link_s = sc.link_s[:0]
    with pytest.raises(LrbmsError):
        ctx_for(sc)
    sc = inputs.custom_scenario(8, 8, 1, 4, 4, 1, 4)
    sc.K = sc.K.copy(); sc.K[3] = -1.0
    with pytest.raises(LrbmsError):
        ctx_for(sc)


def test_rank_deficient_basis_is_numerical_error():
    from paper_1405_2810_b200.lrbms import LrbmsError, LRBMS_E_NUMERICAL
    sc = inputs.custom_scenario(8, 8, 1, 4, 4, 1, 4)
    sc.Phi = sc.Phi.copy()
    sc.Phi[1, 3] = sc.Phi[1, 2]
    ctx = ctx_for(sc)
    with pytest.raises(LrbmsError) as e:
        ctx.run(1)
    assert e.value.status == LRBMS_E_NUMERICAL


@pytest.mark.parametrize("basis", ["pod", "poly"])
@pytest.mark.parametrize("name,steps", [("C2", 100), ("C3", 500)])
def test_full_run_configs(name, steps, basis):
    """Full BASELINE step counts on the paper-recipe bases (pod, the configs as BASELINE states them)
    and on the polynomial bases."""
    sc = inputs.make_scenario(name, basis=basis)
    ref = O.run(sc, n_steps=steps, keep=True)
    ctx = ctx_for(sc)
    dts = np_(ctx.run(steps, log_dt=True))
    s, p, c = ctx.get_state()
    e = dict(dt=rel(dts, ref["dts"]), c=rel(np_(c), ref["cs"][-1]), p=rel(np_(p), ref["ps"][-1]),
             s=float(np.max(np.abs(np_(s) - ref["s"]))))
    print(f"{name} {basis} {steps} steps: " + ", ".join(f"{k} {v:.3e}" for k, v in e.items()))
    assert e["c"] <= 1e-10 and e["p"] <= 1e-10 and e["s"] <= FULL_RUN_S_BAR.get((name, basis), 1e-10)
    assert e["dt"] <= DT_BAR


@pytest.mark.parametrize("name,steps", [("C1", 20), ("C2", 40)])
def test_greedy_bases_run_at_parity(name, steps):
    """Bases from the greedy extension of alg:lrbmsBasisConstruction (offline/recipe.py greedy_recipe:
    true energy-norm error) are one more shared input: the online step on them matches the
    oracle's."""
    sc = inputs.make_scenario(name, basis="greedy")
    ref = O.run(sc, n_steps=steps, keep=True)
    ctx = ctx_for(sc)
    dts = np_(ctx.run(steps, log_dt=True))
    s, p, c = ctx.get_state()
    assert rel(dts, ref["dts"]) <= DT_BAR
    assert rel(np_(c), ref["cs"][-1]) <= 1e-10 and rel(np_(p), ref["ps"][-1]) <= 1e-10
    assert float(np.max(np.abs(np_(s) - ref["s"]))) <= 1e-10


def test_c3_pod_tight_solver():
    """C3 on the paper-recipe bases amplifies round-off (FULL_RUN_S_BAR): with the reduced solve
    iterated to rtol 1e-14 the full 500-step run lands at the level of that amplification."""
    sc = inputs.make_scenario("C3", basis="pod")
    ref = O.run(sc, n_steps=500, keep=True)
    ctx = ctx_for(sc, rtol=1e-14)
    ctx.run(500)
    s, p, c = ctx.get_state()
    ds = float(np.max(np.abs(np_(s) - ref["s"])))
    print(f"C3 pod 500 steps, rtol 1e-14: |ds| {ds:.3e}, rel dc {rel(np_(c), ref['cs'][-1]):.3e}")
    assert rel(np_(c), ref["cs"][-1]) <= 1e-10 and rel(np_(p), ref["ps"][-1]) <= 1e-10
    assert ds <= 3e-10


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_full_size_prefix(name):
    """Full BASELINE sizes in the bench launch configuration: stage parity on s^0 and on a
    random saturation, then a 2-step run against the oracle."""
    sc = inputs.make_scenario(name)
    rng = np.random.default_rng(9)
    s = rng.uniform(0.0, 1.0, sc.n)
    sc.s0 = s
    ctx = ctx_for(sc)
    blocks, r = ctx.stage_project()
    lam = O.total_mobility(s, sc)
    A, b = O.fine_operator(sc, lam)
    ob, orr = O.project(sc, A, b)
    assert rel(np_(blocks), ob) <= 1e-13
    assert rel(np_(r), orr) <= 1e-13
    c = ctx.stage_solve()
    oc = O.solve_reduced(sc, ob, orr)
    assert rel(np_(c), oc) <= 1e-10
    ctx.close()
    sc = inputs.make_scenario(name)
    ref = O.run(sc, n_steps=2, keep=True)
    ctx = ctx_for(sc)
    ctx.run(2)
    sg, pg, cg = ctx.get_state()
    assert rel(np_(cg), ref["cs"][-1]) <= 1e-10
    assert rel(np_(pg), ref["ps"][-1]) <= 1e-10
    assert np.max(np.abs(np_(sg) - ref["s"])) <= 1e-10


GOLDEN_C5 = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "C5_pod_200.npz")


@pytest.mark.parametrize("steps", [10, 200])
def test_c5_golden(steps):
    """The bench workload (C5, paper-recipe bases) in the bench launch configuration against the oracle's
    trajectory written by tests/golden/make_golden.py (oracle only): after 10 and after the full 200
    steps, dt of every step, c and the sampled p within 1e-10 relative, s within 1e-10 absolute.  The
    inputs must be bitwise the golden's (the host recipe is reproducible across hosts, r02b)."""
    import hashlib
    G = np.load(GOLDEN_C5)
    sc = inputs.make_scenario("C5")
    assert hashlib.sha256(np.ascontiguousarray(sc.K).tobytes()).hexdigest() == str(G["K_sha"])
    assert hashlib.sha256(np.ascontiguousarray(sc.Phi).tobytes()).hexdigest() == str(G["Phi_sha"])
    ctx = ctx_for(sc)
    dts = np_(ctx.run(steps, log_dt=True))
    s, p, c = ctx.get_state()
    assert rel(dts, G["dts"][:steps]) <= 1e-10
    assert rel(np_(c), G[f"c_{steps}"]) <= 1e-10
    assert rel(np_(p)[G["cells"]], G[f"p_{steps}"]) <= 1e-10
    assert np.max(np.abs(np_(s) - G[f"s_{steps}"])) <= 1e-10
    ctx.close()


@pytest.mark.parametrize("steps", [20, 50])
def test_c4_prefix_default_solver(steps):
    """C4 (paper-recipe bases) at the product's default solver settings: dt, c and p at the 1e-10 bar
    after 20 and 50 steps, and s at the bar DESIGN.md section 6 derives from C4's measured round-off
    amplification (a 1e-14 input perturbation grows to |ds| ~1e-10 within 50 steps)."""
    sc = inputs.make_scenario("C4")
    ref = O.run(sc, n_steps=steps, keep=True)
    ctx = ctx_for(sc)
    dts = np_(ctx.run(steps, log_dt=True))
    s, p, c = ctx.get_state()
    ds = float(np.max(np.abs(np_(s) - ref["s"])))
    print(f"C4 {steps} steps: |ds| {ds:.3e}, rel dc {rel(np_(c), ref['cs'][-1]):.3e}, "
          f"rel dp {rel(np_(p), ref['ps'][-1]):.3e}")
    assert rel(dts, ref["dts"]) <= DT_BAR
    assert rel(np_(c), ref["cs"][-1]) <= 1e-10
    assert rel(np_(p), ref["ps"][-1]) <= 1e-10
    assert ds <= C4_S_BAR[steps]


def test_c4_prefix_tight_solver():
    """C4 amplifies round-off (a 1e-14 K perturbation gives |ds| 5.7e-11 after 20 steps and 2.2e-6
    after 1000): its saturation parity is checked on a 10-step prefix with a tight
    reduced solve; c and p carry the 1e-10 bar."""
    sc = inputs.make_scenario("C4")
    ref = O.run(sc, n_steps=10, keep=True)
    ctx = ctx_for(sc, rtol=1e-15)
    ctx.run(10)
    s, p, c = ctx.get_state()
    assert rel(np_(c), ref["cs"][-1]) <= 1e-10
    assert rel(np_(p), ref["ps"][-1]) <= 1e-10
    assert np.max(np.abs(np_(s) - ref["s"])) <= 1e-10


# ---------------------------------------------------------------------------- NEXT-1: affine variant

AFFINE = [
    ("C1", lambda: inputs.make_scenario("C1")),
    ("C2", lambda: inputs.make_scenario("C2")),
    # odd n_s (3 x 3) and odd N: the lengths of b_q (9*3*25) and d_q (45) are odd
    ("odd_len", lambda: inputs.custom_scenario(15, 15, 1, 5, 5, 1, 5, seed=26, mu_o=5.0, n_steps=40)),
    ("ragged3d", lambda: inputs.custom_scenario(9, 6, 4, 3, 3, 2, 11, seed=22, mu_o=10.0, bc="corner_columns_3d",
                                                hx=0.5, hy=1.5, hz=2.0, n_steps=40)),
    # round 1's geometric profiles (Euclidean distance instead of the time of flight)
    ("C2_distance", lambda: inputs.make_scenario("C2")),
]


def _profiles(name, sc):
    return inputs.profile_saturations(sc, kind="distance" if name.endswith("_distance") else "tof")


@pytest.mark.parametrize("name,make", AFFINE, ids=[a[0] for a in AFFINE])
def test_affine_stage_parity(name, make):
    """theta fit (as the fitted mobility sum_q theta_q lambda_q, unique even when profiles are
    dependent), the affine reduced system and its solve against the oracle, on a random saturation."""
    sc = make()
    sp = _profiles(name, sc)
    rng = np.random.default_rng(11)
    sc.s0 = rng.uniform(0.0, 1.0, sc.n)
    ctx = ctx_for(sc)
    ctx.set_profiles(sp)
    ctx.set_online(True)
    lq = O.profile_mobilities(sc, sp)
    lam = O.total_mobility(sc.s0, sc)
    th_o = O.theta_fit(sc, lam, lq)
    th_g = np_(ctx.stage_theta())
    fit_o, fit_g = th_o @ lq, th_g @ lq
    assert np.max(np.abs(fit_g - fit_o)) <= 1e-12 * np.max(np.abs(fit_o))
    bq, dq = O.affine_offline(sc, lq)
    ob, orr = O.affine_system(th_o, bq, dq)
    blocks, r = ctx.stage_project()
    assert rel(np_(blocks), ob) <= 1e-12
    assert rel(np_(r), orr) <= 1e-12
    c = ctx.stage_solve()
    oc = O.solve_reduced(sc, ob, orr, method="dense")
    assert rel(np_(c), oc) <= 1e-10


@pytest.mark.parametrize("name,make", AFFINE, ids=[a[0] for a in AFFINE])
def test_affine_full_run(name, make):
    sc = make()
    n = 20
    sp = _profiles(name, sc)
    ref = O.run(sc, n_steps=n, keep=True, s_profiles=sp)
    ctx = ctx_for(sc)
    ctx.set_profiles(sp)
    ctx.set_online(True)
    dts = np_(ctx.run(n, log_dt=True))
    s, p, c = ctx.get_state()
    assert rel(dts, ref["dts"]) <= 1e-10
    assert rel(np_(c), ref["cs"][-1]) <= 1e-10
    assert rel(np_(p), ref["ps"][-1]) <= 1e-10
    assert np.max(np.abs(np_(s) - ref["s"])) <= 1e-10


def test_affine_equals_direct_in_span_gpu():
    """S:556 on the GPU: at a profile's own saturation field the affine reduced system is the direct
    projection (both computed by the library)."""
    sc = inputs.make_scenario("C2")
    sp = inputs.profile_saturations(sc)
    sc.s0 = sp[3].copy()
    ctx = ctx_for(sc)
    bd, rd = (np_(t) for t in ctx.stage_project())
    ctx.set_profiles(sp)
    ctx.set_online(True)
    ba, ra = (np_(t) for t in ctx.stage_project())
    assert rel(ba, bd) <= 1e-12 and rel(ra, rd) <= 1e-12


def test_affine_c5_prefix():
    """The bench workload in the affine variant: 2 steps against the oracle's affine run."""
    sc = inputs.make_scenario("C5")
    sp = inputs.profile_saturations(sc)
    ref = O.run(sc, n_steps=2, keep=True, s_profiles=sp)
    ctx = ctx_for(sc)
    ctx.set_profiles(sp)
    ctx.set_online(True)
    ctx.run(2)
    s, p, c = ctx.get_state()
    assert rel(np_(c), ref["cs"][-1]) <= 1e-10
    assert rel(np_(p), ref["ps"][-1]) <= 1e-10
    assert np.max(np.abs(np_(s) - ref["s"])) <= 1e-10


def test_affine_errors():
    from paper_1405_2810_b200.lrbms import LrbmsError, LRBMS_E_STATE, LRBMS_E_CONFIG
    sc = inputs.make_scenario("C1")
    ctx = ctx_for(sc)
    with pytest.raises(LrbmsError) as e:
        ctx.set_online(True)
    assert e.value.status == LRBMS_E_STATE
    with pytest.raises(LrbmsError) as e:
        ctx.set_profiles(np.zeros((17, sc.n)))
    assert e.value.status == LRBMS_E_CONFIG
    # a new medium or basis invalidates b_q, d_q: the affine variant needs set_profiles again
    sp = inputs.profile_saturations(sc)
    for reset in (lambda: ctx.set_medium(sc.K * 2.0), lambda: ctx.set_basis(sc.Phi)):
        ctx.set_profiles(sp)
        ctx.set_online(True)
        reset()
        with pytest.raises(LrbmsError) as e:
            ctx.set_online(True)
        assert e.value.status == LRBMS_E_STATE


def test_affine_after_new_medium_matches_oracle():
    """set_profiles after set_medium recomputes b_q, d_q with the new K."""
    sc = inputs.make_scenario("C1")
    sp = inputs.profile_saturations(sc)
    ctx = ctx_for(sc)
    ctx.set_profiles(sp)
    sc.K = sc.K * np.linspace(0.5, 2.0, sc.n)
    ctx.set_medium(sc.K)
    ctx.set_profiles(sp)
    ctx.set_online(True)
    ref = O.run(sc, n_steps=5, keep=True, s_profiles=sp)
    ctx.run(5)
    s, p, c = ctx.get_state()
    assert rel(np_(c), ref["cs"][-1]) <= 1e-10
    assert np.max(np.abs(np_(s) - ref["s"])) <= 1e-10
