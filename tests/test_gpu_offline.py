"""NEXT-3: the offline basis recipe on the GPU (lrbms_offline_basis) against the host recipe
(offline/recipe.py, pinned in tests/test_offline_recipe.py) and the oracle's fine operator."""
import numpy as np
import pytest

from offline import recipe as R
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


def projectors(Phi):
    return np.einsum("ekl,ekm->elm", Phi, Phi)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_offline_gpu_matches_host_recipe(name):
    from paper_1405_2810_b200.lrbms import LrbmsContext
    sc = inputs.make_scenario(name, basis="poly")
    seed = 100 + inputs.CONFIG_INDEX[name]
    host = R.pod_recipe(sc, seed, keep_snapshots=True)
    ctx = LrbmsContext(sc)
    Phi, kept, info, tau, snaps = ctx.offline_basis(host.mus, M=8, horizon_steps=sc.n_steps, eps_pca=1e-8,
                                                     rtol=1e-13, want_tau=True, want_snapshots=True)
    Phi, tau, snaps = (t.cpu().numpy() for t in (Phi, tau, snaps))
    print(f"{name}: dt0 {info['dt0']:.6e} (host {host.dt0:.6e}), {info['tof_sweeps']} sweeps, "
          f"{info['fine_cg_iters']} CG iterations, kept {np.bincount(kept)}")
    # Bars.  dt: the pressure error times |p|/|dp| (DT_BAR).  tau divides by the cell's outflow, a sum of
    # pressure differences that is small near stagnation points, and accumulates along the flow paths:
    # the fine pressures' ~1e-12 difference (iterative vs direct solve) is amplified there (max), and adds
    # up over the path length (median; measured 2.9e-11 on C4's 512-cell paths, r02j).  C3 (channels of
    # 1e3..1e4 mD in a 1e-3 background, quarter five-spot) is the ill-conditioned case: the pressures
    # agree to 1.3e-11, but most of its background cells are nearly stagnant (pressure differences of
    # ~1e-8 to their neighbours), so the relative tau difference is ~1e-8 in the median and 8e-6 at the
    # worst cell (r02o / r02q).
    c3 = name == "C3"
    e_tau = np.abs(tau - host.tau) / host.tau
    e_snap = float(np.max(np.abs(snaps - host.P)))
    print(f"  tau: max {e_tau.max():.3e}, median {np.median(e_tau):.3e}; snapshots: max abs {e_snap:.3e}")
    assert info["dt0"] == pytest.approx(host.dt0, rel=1e-8)
    assert e_tau.max() <= (1e-4 if c3 else 1e-7)
    assert np.median(e_tau) <= (1e-7 if c3 else 2e-10)
    # snapshots: against the host's and as solutions of the oracle's independently assembled operator
    assert e_snap <= 1e-10
    lam = host.mus @ (host.LW + host.LO)
    for j in range(0, len(host.mus), max(1, len(host.mus) // 4)):
        A, b = O.fine_operator(sc, lam[j])
        assert np.linalg.norm(b - A @ snaps[j]) <= 1e-10 * np.linalg.norm(b)
    # the bases: orthonormal, indicator first, the same kept modes and the same local spaces
    G = np.einsum("ekl,ejl->ekj", Phi, Phi)
    assert np.max(np.abs(G - np.eye(sc.N)[None])) <= 1e-12
    assert np.max(np.abs(Phi[:, 0, :] - 1.0 / np.sqrt(sc.n_loc))) <= 1e-15
    same = kept == host.kept
    assert same.mean() >= 0.99, (kept[~same], host.kept[~same])
    # the local spaces: the snapshots agree to ~1e-12 (iterative vs direct solves), and a mode with
    # singular value sigma moves by ~ that / sigma; the smallest kept sigma is eps_pca = 1e-8 of the
    # largest, so the projectors may differ by up to ~1e-4 in the weakest kept mode, far less elsewhere
    dP = np.abs(projectors(Phi) - projectors(host.Phi)).max(axis=(1, 2))
    print(f"  projector difference: max {dP[same].max():.3e}, median {np.median(dP[same]):.3e}")
    assert dP[same].max() <= 1e-4 and np.median(dP[same]) <= 1e-6


def test_offline_gpu_basis_runs_at_parity():
    """The GPU-built bases are usable as they are: the online step on them matches the oracle's online
    step on the same bases (c, p at 1e-10, s at 1e-10 after 10 steps)."""
    from paper_1405_2810_b200.lrbms import LrbmsContext
    sc = inputs.make_scenario("C2", basis="poly")
    mus = R.training_parameters(8, 2 * sc.N, 102)
    ctx = LrbmsContext(sc)
    Phi, kept, info, _, _ = ctx.offline_basis(mus, M=8, horizon_steps=sc.n_steps)
    sc.Phi = Phi.cpu().numpy()
    ctx.set_basis(sc.Phi)
    ctx.set_saturation(sc.s0)
    ref = O.run(sc, n_steps=10, keep=True)
    ctx.run(10)
    s, p, c = (t.cpu().numpy() for t in ctx.get_state())
    assert np.max(np.abs(c - ref["cs"][-1])) <= 1e-10 * np.max(np.abs(ref["cs"][-1]))
    assert np.max(np.abs(p - ref["ps"][-1])) <= 1e-10 * np.max(np.abs(ref["ps"][-1]))
    assert np.max(np.abs(s - ref["s"])) <= 1e-10


def test_offline_gpu_errors():
    from paper_1405_2810_b200.lrbms import LrbmsContext, LrbmsError, LRBMS_E_CONFIG
    sc = inputs.make_scenario("C1", basis="poly")
    ctx = LrbmsContext(sc)
    with pytest.raises(LrbmsError) as e:
        ctx.offline_basis(np.full((8, 2), 0.5), M=2)
    assert e.value.status == LRBMS_E_CONFIG
    with pytest.raises(LrbmsError) as e:
        ctx.offline_basis(np.full((65, 8), 1.0 / 8))
    assert e.value.status == LRBMS_E_CONFIG
