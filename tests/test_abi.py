"""The C-ABI library loads and exports every symbol include/lrbms.h declares (CPU only: no
compute calls); host-side validation of lrbms_create works without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lrbms.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1405_2810_b200 import build
    build.build()                      # nvcc cross-compiles for sm_100a without a GPU
    from paper_1405_2810_b200 import lrbms
    return lrbms.load_library()


def header_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lrbms_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    names = header_functions()
    for required in ["lrbms_create", "lrbms_bind", "lrbms_set_medium", "lrbms_set_basis", "lrbms_set_saturation",
                     "lrbms_run", "lrbms_run_host", "lrbms_get_state", "lrbms_stage_project", "lrbms_stage_solve",
                     "lrbms_stage_reconstruct", "lrbms_stage_transport", "lrbms_destroy"]:
        assert required in names


def test_every_declared_symbol_is_exported(lib):
    from paper_1405_2810_b200 import lrbms
    names = header_functions()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(lrbms.EXPORTS) == names          # the binding wraps exactly the declared calls
    assert lib.lrbms_version().decode().startswith("lrbms-b200")


def test_no_undeclared_exports(lib):
    """The product library exports exactly the declared lrbms_* calls (debug hooks only in a
    -DLRBMS_DEBUG build)."""
    import subprocess
    from paper_1405_2810_b200 import build
    out = subprocess.run(["nm", "-D", "--defined-only", build.SO], capture_output=True, text=True).stdout
    exported = sorted({ln.split()[-1] for ln in out.splitlines() if ln.split() and ln.split()[-1].startswith("lrbms_")})
    assert exported == header_functions()


def test_library_targets_sm100a_only():
    from paper_1405_2810_b200 import build
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", build.SO], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", build.SO], capture_output=True, text=True).stdout
    assert "DMMA" in sass            # the projection's fp64 tensor-core path


def _sass_of(prefix):
    """SASS of the kernel whose mangled name starts with ``prefix`` (parameter lists may change)."""
    from paper_1405_2810_b200 import build
    import subprocess
    syms = subprocess.run(["cuobjdump", "-symbols", build.SO], capture_output=True, text=True).stdout.split()
    names = sorted({t for t in syms if t.startswith(prefix)})
    assert names, prefix
    return subprocess.run(["cuobjdump", "-sass", "-fun", names[0], build.SO], capture_output=True, text=True).stdout


def test_onchip_pcg_uses_tensor_memory():
    """k_pcg_tm keeps the scaled couplings in tensor memory: tcgen05.st at staging (STTM), tcgen05.ld
    every iteration (LDTM), cp.async staging (LDGSTS) and release reductions for its grid barriers."""
    sass = _sass_of("_ZN5lrbms8k_pcg_tmILi32ELi448EEE")
    for op in ("LDTM", "STTM", "LDGSTS", "REDG.E.ADD.STRONG.GPU"):
        assert op in sass, op


def test_newton_schulz_on_tcgen05():
    """The coarse inverse's Newton-Schulz GEMM issues tcgen05.mma (UTCHMMA) from TMA-staged tiles."""
    sass = _sass_of("_ZN5lrbms12k_ns_gemm_tcE")
    assert "UTC" in sass and "UTMALDG" in sass


def _create(lib, **over):
    from paper_1405_2810_b200 import lrbms
    import numpy as np
    g = dict(dim=2, nx=16, ny=16, nz=1, hx=1.0, hy=1.0, hz=1.0, sx=8, sy=8, sz=1, N=4)
    g.update(over)
    grid = lrbms.Grid(**g)
    fl = lrbms.Fluid(1.0, 5.0, 0.0, 0.0, 2.0, 2.0)
    cells = np.array([0, 15], np.int32); ax = np.zeros(2, np.int32)
    p = np.array([1.0, 0.0]); s = np.array([1.0, 0.0])
    lk = lrbms.Links(2, cells.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                     ax.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                     p.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                     s.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    h = ctypes.c_void_p()
    st = lib.lrbms_create(ctypes.byref(grid), ctypes.byref(fl), ctypes.byref(lk), ctypes.byref(h))
    return st, h


def test_create_validates_without_gpu(lib):
    st, h = _create(lib)
    assert st == 0 and h
    assert lib.lrbms_workspace_bytes(h) > 0
    # run before bind is a STATE error, not a crash
    assert lib.lrbms_run(h, 1, 0.5, 0.0, None) == 6
    lib.lrbms_destroy(h)
    for bad in [dict(N=33), dict(N=0), dict(sx=5), dict(nz=2), dict(hx=0.0), dict(dim=4)]:
        st, h = _create(lib, **bad)
        assert st == 2, bad
        assert lib.lrbms_last_error(h)
        lib.lrbms_destroy(h)


def test_k1_host_checks_without_gpu(lib):
    """NEXT-4 host logic: N may exceed n_loc up to (dim + 1) n_loc (k = 1 bases), the k = 1 workspace size
    follows the layout, and the k = 1 calls before lrbms_bind are STATE errors, not crashes."""
    st, h = _create(lib, sx=2, sy=2, N=12)          # n_loc = 4, (dim + 1) n_loc = 12
    assert st == 0 and h
    nb = lib.lrbms_k1_bytes(h)
    assert nb >= 8 * (64 * 12 * 3 * 4)                # at least Phi1: n_s N (dim + 1) n_loc doubles
    assert lib.lrbms_k1_run(h, 1, 0.2, 0.0, 1, None) == 6
    assert lib.lrbms_k1_set_saturation(h, None) == 6
    lib.lrbms_destroy(h)
    st, h = _create(lib, sx=2, sy=2, N=13)
    assert st == 2
    lib.lrbms_destroy(h)


def test_onchip_pcg_cluster_mode_in_sass():
    """The mid-size launch of k_pcg_tm synchronises with hardware cluster barriers (UCGABAR / barrier.cluster)."""
    sass = _sass_of("_ZN5lrbms8k_pcg_tmILi0ELi448EEE")
    assert "UCGABAR" in sass or "CGABAR" in sass or "ACQBULK" in sass
