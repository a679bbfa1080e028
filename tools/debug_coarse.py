"""Debug: per-step PCG iterations for the coarse modes, and the accuracy of the device coarse
inverse (||I - E X||) against the device coarse stencil."""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.lrbms import LrbmsContext  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
for mode in (1, 2):
    sc = inputs.make_scenario(cfg)
    ctx = LrbmsContext(sc)
    ctx.set_solver(use_coarse=mode)
    L = ctx.L
    L.lrbms_debug_coarse.restype = ctypes.c_int32
    L.lrbms_debug_coarse.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    n = L.lrbms_debug_coarse(ctx.h, None, None)
    g = sc
    for k in range(steps):
        try:
            ctx.run(1)
        except Exception as e:  # noqa: BLE001
            print(f"mode {mode} step {k}: {e}")
            break
        X = np.zeros((n, n), np.float32)
        Es = np.zeros((sc.n_s, 8))
        L.lrbms_debug_coarse(ctx.h, X.ctypes.data, Es.ctypes.data)
        E = np.eye(n)
        Sx, Sy = sc.Sx, sc.Sy
        Sz = sc.n_s // (Sx * Sy)
        strides = [1, Sx, Sx * Sy]
        dims = [Sx, Sy, Sz]
        for F in range(sc.n_s):
            C = [F % Sx, (F // Sx) % Sy, F // (Sx * Sy)]
            E[F, F] = Es[F, 0]
            for s in range(6):
                a = s % 3
                up = s < 3
                if a >= sc.dim:
                    continue
                if up and C[a] + 1 < dims[a]:
                    E[F, F + strides[a]] = Es[F, 1 + s]
                if (not up) and C[a] > 0:
                    E[F, F - strides[a]] = Es[F, 1 + s]
        asym = np.abs(E - E.T).max()
        rho = np.linalg.norm(np.eye(n) - E @ X.astype(np.float64), 2)
        st = ctx.stats()
        print(f"mode {mode} step {k}: iters {st['last_iters']}, rebuilds {st.get('coarse_rebuilds')}, "
              f"|I - E X| = {rho:.2e}, E asym {asym:.1e}, E diag min {np.diag(E)[:sc.n_s].min():.3e}", flush=True)
