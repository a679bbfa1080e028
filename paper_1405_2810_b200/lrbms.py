"""Thin ctypes binding of liblrbms.so (include/lrbms.h): argument marshalling only.

Every step of the LRBMS online path runs in the library's sm_100a kernels.  PyTorch is
used for device memory (the workspace and the user's tensors) and the CUDA stream.
There is no CPU fallback: if the library or a CUDA device is missing, this raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LRBMS_LIB", os.path.join(HERE, "liblrbms.so"))

LRBMS_OK, LRBMS_E_CONFIG, LRBMS_E_NUMERICAL, LRBMS_E_IO, LRBMS_E_CUDA, LRBMS_E_STATE = 0, 2, 3, 4, 5, 6
STATUS_NAMES = {0: "OK", 2: "CONFIG", 3: "NUMERICAL", 4: "IO", 5: "CUDA", 6: "STATE"}

# Every symbol include/lrbms.h declares (checked by tests/test_abi.py)
EXPORTS = ["lrbms_create", "lrbms_workspace_bytes", "lrbms_bind", "lrbms_set_medium", "lrbms_set_basis",
           "lrbms_set_saturation", "lrbms_set_solver", "lrbms_run", "lrbms_run_host", "lrbms_get_state",
           "lrbms_stage_project", "lrbms_stage_solve", "lrbms_stage_reconstruct", "lrbms_stage_transport",
           "lrbms_get_stats", "lrbms_set_profiling", "lrbms_get_stage_times", "lrbms_launch_count", "lrbms_last_error", "lrbms_version", "lrbms_destroy",
           "lrbms_profiles_bytes", "lrbms_set_profiles", "lrbms_set_online", "lrbms_stage_theta",
           "lrbms_fine_bytes", "lrbms_run_fine", "lrbms_diagnostics", "lrbms_offline_bytes",
           "lrbms_offline_basis", "lrbms_k1_bytes", "lrbms_k1_set_basis", "lrbms_k1_set_saturation",
           "lrbms_k1_run", "lrbms_k1_get_state", "lrbms_k1_stage_project"]


class LrbmsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"lrbms {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Grid(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("hx", ctypes.c_double), ("hy", ctypes.c_double), ("hz", ctypes.c_double),
                ("sx", ctypes.c_int32), ("sy", ctypes.c_int32), ("sz", ctypes.c_int32), ("N", ctypes.c_int32)]


class Fluid(ctypes.Structure):
    _fields_ = [("mu_w", ctypes.c_double), ("mu_o", ctypes.c_double), ("swr", ctypes.c_double),
                ("sor", ctypes.c_double), ("nw", ctypes.c_double), ("no", ctypes.c_double)]


class Links(ctypes.Structure):
    _fields_ = [("n_links", ctypes.c_int32), ("cell", ctypes.POINTER(ctypes.c_int32)),
                ("axis", ctypes.POINTER(ctypes.c_int32)), ("p", ctypes.POINTER(ctypes.c_double)),
                ("s_ext", ctypes.POINTER(ctypes.c_double))]


class SolverOpts(ctypes.Structure):
    _fields_ = [("rtol", ctypes.c_double), ("max_iters", ctypes.c_int32), ("coarse_refresh", ctypes.c_int32),
                ("use_coarse", ctypes.c_int32), ("history", ctypes.c_int32),
                ("onchip", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_int64), ("t", ctypes.c_double), ("last_dt", ctypes.c_double),
                ("last_iters", ctypes.c_int32), ("total_iters", ctypes.c_int64),
                ("coarse_rebuilds", ctypes.c_int32), ("fprime_max", ctypes.c_double),
                ("ns_guard_trips", ctypes.c_int64), ("ns_resid_max", ctypes.c_double)]


class OfflineInfo(ctypes.Structure):
    _fields_ = [("dt0", ctypes.c_double), ("horizon", ctypes.c_double), ("tof_sweeps", ctypes.c_int32),
                ("fine_cg_iters", ctypes.c_int64)]


class Diag(ctypes.Structure):
    _fields_ = [(k, ctypes.c_double) for k in ("mass_prev", "mass", "s_min", "s_max", "zeta_max", "zeta_mean",
                                               "coarse_defect", "water_out", "q_in", "q_out", "dt", "mass_balance")]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load liblrbms.so (fails loudly; build it with paper_1405_2810_b200/build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"liblrbms.so not found at {path}: run `python -m paper_1405_2810_b200.build` "
                           "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    P = ctypes.c_void_p
    D = ctypes.c_double
    I = ctypes.c_int32
    st = ctypes.c_int
    sig = {
        "lrbms_create": (st, [ctypes.POINTER(Grid), ctypes.POINTER(Fluid), ctypes.POINTER(Links), ctypes.POINTER(P)]),
        "lrbms_workspace_bytes": (ctypes.c_size_t, [P]),
        "lrbms_bind": (st, [P, P, ctypes.c_size_t, P]),
        "lrbms_set_medium": (st, [P, P, P]),
        "lrbms_set_basis": (st, [P, P]),
        "lrbms_set_saturation": (st, [P, P]),
        "lrbms_set_solver": (st, [P, ctypes.POINTER(SolverOpts)]),
        "lrbms_run": (st, [P, I, D, D, P]),
        "lrbms_run_host": (st, [P, I, D, D, P, P, P]),
        "lrbms_get_state": (st, [P, P, P, P]),
        "lrbms_stage_project": (st, [P, P, P]),
        "lrbms_stage_solve": (st, [P, P]),
        "lrbms_stage_reconstruct": (st, [P, P]),
        "lrbms_stage_transport": (st, [P, D, D, P, P, P]),
        "lrbms_get_stats": (st, [P, ctypes.POINTER(Stats)]),
        "lrbms_launch_count": (ctypes.c_int64, [P]),
        "lrbms_set_profiling": (st, [P, I]),
        "lrbms_profiles_bytes": (ctypes.c_size_t, [P, I]),
        "lrbms_set_profiles": (st, [P, P, I, P, ctypes.c_size_t]),
        "lrbms_set_online": (st, [P, I]),
        "lrbms_stage_theta": (st, [P, P]),
        "lrbms_fine_bytes": (ctypes.c_size_t, [P]),
        "lrbms_run_fine": (st, [P, I, D, D, P, P, ctypes.c_size_t, D, I, ctypes.POINTER(ctypes.c_int64)]),
        "lrbms_diagnostics": (st, [P, ctypes.POINTER(Diag)]),
        "lrbms_offline_bytes": (ctypes.c_size_t, [P, I]),
        "lrbms_offline_basis": (st, [P, I, I, P, I, D, D, D, P, ctypes.c_size_t, P, P, P, P,
                                     ctypes.POINTER(OfflineInfo)]),
        "lrbms_k1_bytes": (ctypes.c_size_t, [P]),
        "lrbms_k1_set_basis": (st, [P, P, D, P, ctypes.c_size_t]),
        "lrbms_k1_set_saturation": (st, [P, P]),
        "lrbms_k1_run": (st, [P, I, D, D, I, P]),
        "lrbms_k1_get_state": (st, [P, P, P, P, ctypes.POINTER(ctypes.c_int32)]),
        "lrbms_k1_stage_project": (st, [P, P, P]),
        "lrbms_get_stage_times": (st, [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64), I]),
        "lrbms_last_error": (ctypes.c_char_p, [P]),
        "lrbms_version": (ctypes.c_char_p, []),
        "lrbms_destroy": (None, [P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


class LrbmsContext:
    """One LRBMS online problem on one GPU (wraps lrbms_ctx).

    ``sc`` is a scenario with the fields of paper_1405_2810_b200.inputs.Scenario: grid and
    partition sizes, fluid constants, links (cell, axis, p, s_ext), K, phi, Phi, s0.
    """

    def __init__(self, sc, device="cuda", stream=None, solver: Optional[dict] = None, k1_only: bool = False):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("LrbmsContext needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.L = load_library()
        self.sc = sc
        self.device = torch.device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        g = Grid(sc.dim, sc.nx, sc.ny, sc.nz, sc.hx, sc.hy, sc.hz, sc.sx, sc.sy, sc.sz, sc.N)
        f = Fluid(sc.mu_w, sc.mu_o, sc.swr, sc.sor, sc.nw, sc.no)
        self._lk = [np.ascontiguousarray(sc.link_cell, np.int32), np.ascontiguousarray(sc.link_axis, np.int32),
                    np.ascontiguousarray(sc.link_p, np.float64), np.ascontiguousarray(sc.link_s, np.float64)]
        lk = Links(len(self._lk[0]),
                   self._lk[0].ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                   self._lk[1].ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                   self._lk[2].ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                   self._lk[3].ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        h = ctypes.c_void_p()
        status = self.L.lrbms_create(ctypes.byref(g), ctypes.byref(f), ctypes.byref(lk), ctypes.byref(h))
        self.h = h
        if status != LRBMS_OK:
            msg = self.L.lrbms_last_error(h).decode() if h else "create failed"
            if h:
                self.L.lrbms_destroy(h)
                self.h = None
            raise LrbmsError(status, msg)
        nbytes = self.L.lrbms_workspace_bytes(h)
        with torch.cuda.device(self.device):
            self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        base = self.workspace.data_ptr()
        self._ws_ptr = (base + 255) // 256 * 256
        self._check(self.L.lrbms_bind(h, ctypes.c_void_p(self._ws_ptr), nbytes,
                                      ctypes.c_void_p(self.stream.cuda_stream)))
        if solver:
            self.set_solver(**solver)
        self.set_medium(sc.K, sc.phi)
        if not k1_only:   # k1_only: a context for the k = 1 fine space alone (NEXT-4; N may exceed n_loc)
            self.set_basis(sc.Phi)
            self.set_saturation(sc.s0)

    # -- helpers -----------------------------------------------------------------------------
    def _check(self, status):
        if status != LRBMS_OK:
            raise LrbmsError(status, self.L.lrbms_last_error(self.h).decode())

    def dev(self, a, dtype=None):
        torch = self.torch
        dtype = dtype or torch.float64
        if isinstance(a, torch.Tensor):
            return a.to(device=self.device, dtype=dtype).contiguous()
        return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=self.device)

    def empty(self, *shape):
        return self.torch.empty(*shape, dtype=self.torch.float64, device=self.device)

    # -- API ---------------------------------------------------------------------------------
    def set_medium(self, K, phi=None):
        self._K = self.dev(K)
        self._phi = None if phi is None else self.dev(phi)
        self._check(self.L.lrbms_set_medium(self.h, _ptr(self._K), _ptr(self._phi)))

    def set_basis(self, Phi):
        self._Phi = self.dev(Phi)
        self._check(self.L.lrbms_set_basis(self.h, _ptr(self._Phi)))
        self.stream.synchronize()
        self._Phi = None

    def set_saturation(self, s):
        t = self.dev(s)
        self._check(self.L.lrbms_set_saturation(self.h, _ptr(t)))
        self.stream.synchronize()

    def set_solver(self, rtol=5e-13, max_iters=5000, coarse_refresh=200, use_coarse=2, history=8, onchip=1):
        o = SolverOpts(rtol, max_iters, coarse_refresh, use_coarse, history, onchip)
        self._check(self.L.lrbms_set_solver(self.h, ctypes.byref(o)))

    def run(self, n_steps, cfl=None, dt_fixed=0.0, log_dt=False):
        cfl = self.sc.cfl if cfl is None else cfl
        dt_log = self.empty(max(n_steps, 1)) if log_dt else None
        self._check(self.L.lrbms_run(self.h, int(n_steps), float(cfl), float(dt_fixed), _ptr(dt_log)))
        return dt_log[:n_steps] if log_dt else None

    def run_host(self, n_steps, s_in=None, cfl=None, dt_fixed=0.0, want_s=True, want_p=False):
        """End-to-end from host buffers (the e2e path): returns numpy (s, p)."""
        cfl = self.sc.cfl if cfl is None else cfl
        n = self.sc.n
        s_out = np.empty(n) if want_s else None
        p_out = np.empty(n) if want_p else None
        sp = None
        if s_in is not None:
            s_in = np.ascontiguousarray(s_in, np.float64)
            sp = s_in.ctypes.data_as(ctypes.c_void_p)
        self._check(self.L.lrbms_run_host(self.h, int(n_steps), float(cfl), float(dt_fixed), sp,
                                          None if s_out is None else s_out.ctypes.data_as(ctypes.c_void_p),
                                          None if p_out is None else p_out.ctypes.data_as(ctypes.c_void_p)))
        return s_out, p_out

    def run_host_ptr(self, n_steps, s_in_ptr, s_out_ptr, p_out_ptr=None, cfl=None, dt_fixed=0.0):
        """e2e with caller-owned (e.g. pinned) host buffers given as integer addresses."""
        cfl = self.sc.cfl if cfl is None else cfl
        c = lambda v: None if v is None else ctypes.c_void_p(v)
        self._check(self.L.lrbms_run_host(self.h, int(n_steps), float(cfl), float(dt_fixed), c(s_in_ptr),
                                          c(s_out_ptr), c(p_out_ptr)))

    def get_state(self):
        sc = self.sc
        s, p, c = self.empty(sc.n), self.empty(sc.n), self.empty(sc.n_s * sc.N)
        self._check(self.L.lrbms_get_state(self.h, _ptr(s), _ptr(p), _ptr(c)))
        return s, p, c.view(sc.n_s, sc.N)

    def set_profiles(self, s_profiles):
        """NEXT-1: the M profile saturation fields ([M][n], natural order) of the paper's affine online
        variant; allocates the caller-owned profile workspace (marshalling only)."""
        torch = self.torch
        sp = np.ascontiguousarray(s_profiles, np.float64)
        M = int(sp.shape[0])
        nbytes = self.L.lrbms_profiles_bytes(self.h, M)
        if nbytes == 0:
            raise LrbmsError(LRBMS_E_CONFIG, f"number of profiles M = {M} not supported")
        with torch.cuda.device(self.device):
            self.profile_ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        ptr = (self.profile_ws.data_ptr() + 255) // 256 * 256
        self._profiles_dev = self.dev(sp.reshape(M, -1))
        self.n_profiles = M
        self._check(self.L.lrbms_set_profiles(self.h, _ptr(self._profiles_dev), M, ctypes.c_void_p(ptr), nbytes))

    def run_fine(self, n_steps, cfl=None, dt_fixed=0.0, log_dt=False, rtol=1e-12, max_iters=100000):
        """NEXT-2: n_steps of the fine-scale reference scheme (Phi_E = I; lrbms_run_fine) from the
        current state; allocates the caller-owned fine workspace once (marshalling only).
        Returns (dt_log or None, CG iterations summed over the steps)."""
        torch = self.torch
        cfl = self.sc.cfl if cfl is None else cfl
        nbytes = self.L.lrbms_fine_bytes(self.h)
        if getattr(self, "fine_ws", None) is None or self.fine_ws.numel() < nbytes + 256:
            with torch.cuda.device(self.device):
                self.fine_ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        ptr = (self.fine_ws.data_ptr() + 255) // 256 * 256
        dt_log = self.empty(max(n_steps, 1)) if log_dt else None
        iters = ctypes.c_int64(0)
        self._check(self.L.lrbms_run_fine(self.h, int(n_steps), float(cfl), float(dt_fixed), _ptr(dt_log),
                                          ctypes.c_void_p(ptr), nbytes, float(rtol), int(max_iters),
                                          ctypes.byref(iters)))
        return (dt_log[:n_steps] if log_dt else None), int(iters.value)

    def set_online(self, affine: bool):
        self._check(self.L.lrbms_set_online(self.h, 1 if affine else 0))

    def stage_theta(self):
        th = self.empty(self.n_profiles)
        self._check(self.L.lrbms_stage_theta(self.h, _ptr(th)))
        return th

    def stage_project(self):
        sc = self.sc
        blocks = self.empty(sc.n_s, 1 + sc.dim, sc.N, sc.N)
        r = self.empty(sc.n_s, sc.N)
        self._check(self.L.lrbms_stage_project(self.h, _ptr(blocks), _ptr(r)))
        return blocks, r

    def stage_solve(self):
        c = self.empty(self.sc.n_s, self.sc.N)
        self._check(self.L.lrbms_stage_solve(self.h, _ptr(c)))
        return c

    def stage_reconstruct(self):
        p = self.empty(self.sc.n)
        self._check(self.L.lrbms_stage_reconstruct(self.h, _ptr(p)))
        return p

    def n_interior_faces(self):
        sc = self.sc
        return (sc.nx - 1) * sc.ny * sc.nz + sc.nx * (sc.ny - 1) * sc.nz + sc.nx * sc.ny * (sc.nz - 1)

    def stage_transport(self, cfl=None, dt_fixed=0.0):
        cfl = self.sc.cfl if cfl is None else cfl
        ff = self.empty(max(self.n_interior_faces(), 1))
        lf = self.empty(max(self.sc.n_links, 1))
        dt = self.empty(1)
        self._check(self.L.lrbms_stage_transport(self.h, float(cfl), float(dt_fixed), _ptr(ff), _ptr(lf), _ptr(dt)))
        return ff[:self.n_interior_faces()], lf[:self.sc.n_links], dt

    def stats(self) -> dict:
        st = Stats()
        self._check(self.L.lrbms_get_stats(self.h, ctypes.byref(st)))
        return {k: getattr(st, k) for k, _ in Stats._fields_}

    def offline_basis(self, mus, M=8, horizon_steps=None, cfl=None, eps_pca=1e-8, rtol=1e-13,
                      want_tau=False, want_snapshots=False):
        """NEXT-3: the offline basis recipe on the GPU (lrbms_offline_basis) from the current saturation;
        mus: [n_train][M] training parameters (host).  Returns (Phi [n_s][N][n_loc] device tensor,
        kept (numpy), info dict, tau or None, snapshots or None).  Marshalling only."""
        torch = self.torch
        sc = self.sc
        mus = np.ascontiguousarray(mus, np.float64)
        J = int(mus.shape[0])
        nbytes = self.L.lrbms_offline_bytes(self.h, J)
        if nbytes == 0:
            raise LrbmsError(LRBMS_E_CONFIG, f"n_train = {J} not supported")
        with torch.cuda.device(self.device):
            ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        ptr = (ws.data_ptr() + 255) // 256 * 256
        Phi = self.empty(sc.n_s, sc.N, sc.n_loc)
        tau = self.empty(sc.n) if want_tau else None
        snaps = self.empty(J, sc.n) if want_snapshots else None
        kept = np.zeros(sc.n_s, np.int32)
        info = OfflineInfo()
        hs = sc.n_steps if horizon_steps is None else horizon_steps
        self._check(self.L.lrbms_offline_basis(
            self.h, int(M), J, mus.ctypes.data_as(ctypes.c_void_p), int(hs), float(sc.cfl if cfl is None else cfl),
            float(eps_pca), float(rtol), ctypes.c_void_p(ptr), nbytes, _ptr(Phi), _ptr(tau), _ptr(snaps),
            kept.ctypes.data_as(ctypes.c_void_p), ctypes.byref(info)))
        del ws
        return Phi, kept, {k: getattr(info, k) for k, _ in OfflineInfo._fields_}, tau, snaps

    # -- NEXT-4: the k = 1 fine space (marshalling only) ----------------------------------------
    def k1_set_basis(self, Phi1, c_pen=None):
        torch = self.torch
        sc = self.sc
        nbytes = self.L.lrbms_k1_bytes(self.h)
        with torch.cuda.device(self.device):
            self.k1_ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        ptr = (self.k1_ws.data_ptr() + 255) // 256 * 256
        t = self.dev(Phi1)
        assert t.numel() == sc.n_s * sc.N * (sc.dim + 1) * sc.n_loc, "Phi1 must be [n_s][N][(dim + 1) n_loc]"
        self._check(self.L.lrbms_k1_set_basis(self.h, _ptr(t), float(sc.c_pen if c_pen is None else c_pen),
                                              ctypes.c_void_p(ptr), nbytes))

    def k1_set_saturation(self, s1):
        t = self.dev(np.asarray(s1, np.float64).reshape(self.sc.dim + 1, self.sc.n))
        self._check(self.L.lrbms_k1_set_saturation(self.h, _ptr(t)))
        self.stream.synchronize()

    def k1_run(self, n_steps, cfl=None, dt_fixed=0.0, limiter=True, log_dt=False):
        cfl = self.sc.cfl if cfl is None else cfl
        dt_log = self.empty(max(n_steps, 1)) if log_dt else None
        self._check(self.L.lrbms_k1_run(self.h, int(n_steps), float(cfl), float(dt_fixed), 1 if limiter else 0,
                                        _ptr(dt_log)))
        return dt_log[:n_steps] if log_dt else None

    def k1_get_state(self):
        sc = self.sc
        nd = sc.dim + 1
        s1, p1, c = self.empty(nd, sc.n), self.empty(nd, sc.n), self.empty(sc.n_s, sc.N)
        nf = ctypes.c_int32(0)
        self._check(self.L.lrbms_k1_get_state(self.h, _ptr(s1), _ptr(p1), _ptr(c), ctypes.byref(nf)))
        return s1, p1, c, int(nf.value)

    def k1_stage_project(self):
        sc = self.sc
        blocks = self.empty(sc.n_s, 1 + sc.dim, sc.N, sc.N)
        r = self.empty(sc.n_s, sc.N)
        self._check(self.L.lrbms_k1_stage_project(self.h, _ptr(blocks), _ptr(r)))
        return blocks, r

    def diagnostics(self) -> dict:
        """K6 diagnostics of the last step (lrbms_diagnostics): mass, s range, zeta, coarse defect."""
        d = Diag()
        self._check(self.L.lrbms_diagnostics(self.h, ctypes.byref(d)))
        return {k: getattr(d, k) for k, _ in Diag._fields_}

    STAGES = ["project", "coarse", "scale", "guess", "pcg", "recon", "flux_cfl", "transport"]

    def set_profiling(self, on: bool):
        self._check(self.L.lrbms_set_profiling(self.h, 1 if on else 0))

    def stage_times(self) -> dict:
        n = len(self.STAGES)
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        self._check(self.L.lrbms_get_stage_times(self.h, ms, cnt, n))
        return {name: (ms[i], cnt[i]) for i, name in enumerate(self.STAGES)}

    def launch_count(self) -> int:
        return int(self.L.lrbms_launch_count(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.L.lrbms_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
