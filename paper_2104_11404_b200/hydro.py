"""Thin ctypes binding of include/hydro.h (argument marshalling only).

Every step of the hot path runs in libhydro.so's CUDA kernels; this module only
passes torch tensors' device pointers and the current CUDA stream.  There is no
CPU fallback: if the library is missing or no CUDA device is present, calls
raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# HYDRO_LIB_PATH: load another in-tree build of the same library (A/B of kernel variants,
# tools/ab_lib.py); never a substitute implementation.
LIB_PATH = os.environ.get("HYDRO_LIB_PATH") or os.path.join(_HERE, "libhydro.so")

HYDRO_OK, HYDRO_ERR_ARG, HYDRO_ERR_UNSUPPORTED, HYDRO_ERR_CUDA = 0, 1, 2, 3
HYDRO_ERR_TANGLED, HYDRO_ERR_NONFINITE, HYDRO_ERR_WORKSPACE, HYDRO_ERR_NOT_CONVERGED = 4, 5, 6, 7
STATUS_NAMES = {0: "OK", 1: "ERR_ARG", 2: "ERR_UNSUPPORTED", 3: "ERR_CUDA", 4: "ERR_TANGLED",
                5: "ERR_NONFINITE", 6: "ERR_WORKSPACE", 7: "ERR_NOT_CONVERGED"}

EXPORTED = ["hydro_ctx_workspace_bytes", "hydro_ctx_create", "hydro_ctx_destroy",
            "hydro_force_full", "hydro_dt_estimate", "hydro_status_sync", "hydro_sample_create",
            "hydro_sample_destroy", "hydro_sample_info", "hydro_sample_lists", "hydro_rom_lift",
            "hydro_force_sampled", "hydro_sample_status_sync", "hydro_rom_project_workspace_bytes",
            "hydro_rom_project", "hydro_basis_tables", "hydro_launch_count", "hydro_version", "hydro_set_2d_kernel",
            "hydro_profile_enable", "hydro_profile_read", "hydro_profile_read_captured",
            "hydro_profile_release_captured", "hydro_selftest_ieee_fast",
            "hydro_fom_create", "hydro_fom_destroy", "hydro_mass_v_apply", "hydro_mass_v_solve",
            "hydro_mass_e_solve", "hydro_fom_energy", "hydro_rk2avg_step", "hydro_fom_advance", "hydro_rom_advance", "hydro_rom_create",
            "hydro_fom_stage_state", "hydro_pod", "hydro_deim", "hydro_qdeim", "hydro_deim_oversampled", "hydro_mass_e_apply", "hydro_window_ops", "hydro_gappy_pinv", "hydro_rom_window_offset", "hydro_basis_tproduct", "hydro_rom_indicator", "hydro_index_copy_add",
            "hydro_rom_destroy", "hydro_rom_rk2avg_step", "hydro_force_stress_bytes",
            "hydro_force_full_store", "hydro_force_transpose", "hydro_sample_stress_bytes",
            "hydro_force_sampled_store", "hydro_sample_force_transpose"]


class HydroError(RuntimeError):
    def __init__(self, code: int, what: str, first_bad: int = -1):
        super().__init__(f"{what}: {STATUS_NAMES.get(code, code)}"
                         + (f" (first tangled element {first_bad})" if first_bad >= 0 else ""))
        self.code = code
        self.first_bad = first_bad


class _MeshDesc(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("order_h1", ctypes.c_int), ("nq1d", ctypes.c_int),
                ("n_elem", ctypes.c_int64), ("n_nodes", ctypes.c_int64),
                ("elem_nodes", ctypes.c_void_p), ("x0", ctypes.c_void_p), ("rho0", ctypes.c_void_p)]


class _Visc(ctypes.Structure):
    _fields_ = [("q1", ctypes.c_double), ("q2", ctypes.c_double), ("enabled", ctypes.c_int)]


class _Cfl(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("alpha_mu", ctypes.c_double)]


class _DtCtrl(ctypes.Structure):
    _fields_ = [("beta1", ctypes.c_double), ("beta2", ctypes.c_double), ("gamma", ctypes.c_double)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libhydro.so (built in-tree by paper_2104_11404_b200.build). Raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2104_11404_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.hydro_ctx_workspace_bytes.restype = ctypes.c_size_t
        L.hydro_ctx_workspace_bytes.argtypes = [ctypes.POINTER(_MeshDesc)]
        L.hydro_ctx_create.argtypes = [ctypes.POINTER(_MeshDesc), vp, ctypes.c_size_t, vp,
                                       ctypes.POINTER(vp)]
        L.hydro_ctx_destroy.argtypes = [vp]
        L.hydro_force_full.argtypes = [vp, vp, vp, vp, vp, vp, _Visc, _Cfl, vp, vp, vp, vp]
        L.hydro_dt_estimate.argtypes = [vp, vp, vp, vp, vp, _Visc, _Cfl, vp, vp]
        L.hydro_status_sync.argtypes = [vp, vp, ctypes.POINTER(i64)]
        L.hydro_sample_create.argtypes = [vp, vp, i64, i32, ctypes.POINTER(vp)]
        L.hydro_sample_destroy.argtypes = [vp]
        L.hydro_sample_info.argtypes = [vp] + [ctypes.POINTER(i64)] * 5
        L.hydro_sample_lists.argtypes = [vp, vp, vp, vp]
        L.hydro_rom_lift.argtypes = [i64, i32, i32, vp, vp, i32, vp, vp, vp]
        L.hydro_force_sampled.argtypes = [vp, vp, vp, vp, vp, vp, _Visc, _Cfl, vp, vp, vp, vp]
        L.hydro_sample_status_sync.argtypes = [vp, vp, ctypes.POINTER(i64)]
        L.hydro_selftest_ieee_fast.argtypes = [ctypes.c_uint64, i64, i32, i32, vp, vp]
        L.hydro_fom_create.argtypes = [vp, vp, i64, vp, ctypes.POINTER(vp)]
        L.hydro_fom_destroy.argtypes = [vp]
        L.hydro_mass_v_apply.argtypes = [vp, vp, vp, vp]
        L.hydro_mass_v_solve.argtypes = [vp, vp, vp, dbl, i32, ctypes.POINTER(i32),
                                         ctypes.POINTER(dbl), vp]
        L.hydro_mass_e_solve.argtypes = [vp, vp, vp, vp]
        L.hydro_mass_e_apply.argtypes = [vp, vp, vp, vp]
        L.hydro_window_ops.argtypes = [vp, i32, i64, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp]
        L.hydro_gappy_pinv.argtypes = [vp, i64, i32, ctypes.POINTER(i64), i64, vp, vp]
        L.hydro_rom_window_offset.argtypes = [i64, i32, i32, vp, vp, i32, vp, vp, i32, vp, vp]
        L.hydro_basis_tproduct.argtypes = [i64, i32, i32, vp, vp, vp, vp]
        L.hydro_index_copy_add.argtypes = [i64, i32, vp, i64, vp, vp, i64, vp, i32, vp]
        L.hydro_rom_indicator.argtypes = [vp, vp, vp, vp, vp, _Visc, _Cfl, i32, vp, i32, vp, i32, vp, i32,
                                          ctypes.POINTER(i64), i32, vp, i32, ctypes.POINTER(i64),
                                          ctypes.POINTER(ctypes.c_double), vp]
        L.hydro_fom_energy.argtypes = [vp, vp, vp, ctypes.POINTER(dbl), ctypes.POINTER(dbl), vp]
        L.hydro_rk2avg_step.argtypes = [vp, vp, vp, vp, vp, _Visc, _Cfl, dbl, dbl, i32,
                                        ctypes.POINTER(dbl), ctypes.POINTER(i32), vp]
        L.hydro_fom_advance.argtypes = [vp, vp, vp, vp, vp, _Visc, _Cfl, _DtCtrl, dbl, dbl,
                                        ctypes.POINTER(dbl), i32, dbl, i32, ctypes.POINTER(dbl),
                                        ctypes.POINTER(i32), ctypes.POINTER(i32), vp]
        L.hydro_rom_create.argtypes = [vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, i32, vp, vp, vp,
                                       vp, ctypes.POINTER(vp)]
        L.hydro_rom_destroy.argtypes = [vp]
        L.hydro_rom_rk2avg_step.argtypes = [vp, vp, vp, vp, vp, _Visc, _Cfl, vp, vp, vp]
        L.hydro_fom_stage_state.argtypes = [vp, vp, vp, vp, vp]
        L.hydro_pod.argtypes = [vp, i32, i64, dbl, i32, vp, ctypes.POINTER(dbl),
                                ctypes.POINTER(i32), vp]
        L.hydro_deim.argtypes = [vp, i64, i32, ctypes.POINTER(i64), vp]
        L.hydro_qdeim.argtypes = [vp, i64, i32, ctypes.POINTER(i64), vp]
        L.hydro_deim_oversampled.argtypes = [vp, i64, i32, i32, ctypes.POINTER(i64), vp]
        L.hydro_rom_advance.argtypes = [vp, vp, vp, vp, vp, _Visc, _Cfl, _DtCtrl, dbl, dbl,
                                        ctypes.POINTER(dbl), i32, ctypes.POINTER(dbl),
                                        ctypes.POINTER(i32), ctypes.POINTER(i32),
                                        ctypes.POINTER(i32), vp]
        L.hydro_force_stress_bytes.restype = ctypes.c_size_t
        L.hydro_force_stress_bytes.argtypes = [vp]
        L.hydro_force_full_store.argtypes = [vp, vp, vp, vp, vp, _Visc, _Cfl, vp, vp, vp, vp, vp]
        L.hydro_force_transpose.argtypes = [vp, vp, vp, vp, vp]
        L.hydro_sample_stress_bytes.restype = ctypes.c_size_t
        L.hydro_sample_stress_bytes.argtypes = [vp]
        L.hydro_force_sampled_store.argtypes = [vp, vp, vp, vp, vp, _Visc, _Cfl, vp, vp, vp, vp, vp]
        L.hydro_sample_force_transpose.argtypes = [vp, vp, vp, vp, vp]
        L.hydro_rom_project_workspace_bytes.restype = ctypes.c_size_t
        L.hydro_rom_project_workspace_bytes.argtypes = [i32, i64, i32]
        L.hydro_rom_project.argtypes = [i32, i64, i32, vp, vp, vp, vp, ctypes.c_size_t, vp]
        L.hydro_basis_tables.argtypes = [i32, i32, vp, vp, vp, vp, vp]
        L.hydro_launch_count.restype = i64
        L.hydro_profile_enable.argtypes = [i32]
        L.hydro_profile_read.argtypes = [ctypes.POINTER(dbl), ctypes.POINTER(i64)]
        L.hydro_profile_read_captured.argtypes = [ctypes.POINTER(dbl), ctypes.POINTER(i64)]
        L.hydro_profile_release_captured.argtypes = []
        L.hydro_version.restype = ctypes.c_char_p
        L.hydro_set_2d_kernel.argtypes = [i32]
        _lib = L
    return _lib


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("hydro: tensors must live on the CUDA device")
    if t.dtype not in (torch.float64, torch.int32, torch.int64, torch.uint8):
        raise ValueError(f"hydro: unexpected dtype {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("hydro: tensors must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream: Optional[torch.cuda.Stream] = None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _check(rc: int, what: str):
    if rc != HYDRO_OK:
        raise HydroError(rc, what)


@dataclass
class Visc:
    q1: float = 0.5
    q2: float = 2.0
    enabled: bool = True

    def c(self):
        return _Visc(self.q1, self.q2, 1 if self.enabled else 0)


@dataclass
class Cfl:
    alpha: float = 0.5
    alpha_mu: float = 2.5

    def c(self):
        return _Cfl(self.alpha, self.alpha_mu)


@dataclass
class DtCtrl:
    """Time-step controller constants (PAPER P:549-566 defaults)."""
    beta1: float = 0.85
    beta2: float = 1.02
    gamma: float = 0.8

    def c(self):
        return _DtCtrl(self.beta1, self.beta2, self.gamma)


def basis_tables(k: int, q: int) -> dict:
    """The library's own correctly rounded tables (host computation)."""
    import numpy as np
    xi, w = np.zeros(q), np.zeros(q)
    B, G, Bl = np.zeros((q, k + 1)), np.zeros((q, k + 1)), np.zeros((q, k))
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    _check(lib().hydro_basis_tables(k, q, p(xi), p(w), p(B), p(G), p(Bl)), "hydro_basis_tables")
    return dict(xi=xi, w=w, B=B, G=G, Bl=Bl)


def selftest_ieee_fast(seed: int, n: int, op: int, dist: int, stream=None):
    """(mismatches, slow-path operands, total) of the fast div/rcp/sqrt paths vs IEEE."""
    counts = torch.zeros(3, dtype=torch.int64, device="cuda")
    _check(lib().hydro_selftest_ieee_fast(seed, n, op, dist, _ptr(counts), _stream(stream)),
           "hydro_selftest_ieee_fast")
    return tuple(int(x) for x in counts.cpu().tolist())


_K2D = {"auto": 0, "element": 1, "point": 2, "lane": 3}


def set_kernel_2d(choice: str) -> None:
    """hydro_set_2d_kernel: "auto" (by size), "element" (one thread per element), "point" (one
    thread per point, generic kernel) or "lane" (one lane per point, q1 per warp)."""
    _check(lib().hydro_set_2d_kernel(_K2D[choice]), "hydro_set_2d_kernel")


def launch_count() -> int:
    return int(lib().hydro_launch_count())


def profile_enable(on: bool = True) -> None:
    _check(lib().hydro_profile_enable(1 if on else 0), "hydro_profile_enable")


def profile_read():
    """(summed force-kernel ms, launches) since the last read; synchronises."""
    ms, n = ctypes.c_double(0.0), ctypes.c_int64(0)
    _check(lib().hydro_profile_read(ctypes.byref(ms), ctypes.byref(n)), "hydro_profile_read")
    return ms.value, n.value


def profile_read_captured():
    """(summed force-kernel ms, launches) of the most recent replay of a graph captured with
    profiling enabled (the events stay attached to the graph)."""
    ms, n = ctypes.c_double(0.0), ctypes.c_int64(0)
    _check(lib().hydro_profile_read_captured(ctypes.byref(ms), ctypes.byref(n)),
           "hydro_profile_read_captured")
    return ms.value, n.value


def profile_release_captured() -> None:
    _check(lib().hydro_profile_release_captured(), "hydro_profile_release_captured")


class HydroContext:
    """Mesh context (hydro_ctx_create): m_q, assembly slots, dt status in a torch workspace."""

    def __init__(self, dim: int, k: int, nq: int, elem_nodes: torch.Tensor, x0: torch.Tensor,
                 rho0: torch.Tensor, stream: Optional[torch.cuda.Stream] = None):
        L = lib()
        self.dim, self.k, self.nq = dim, k, nq
        self.elem_nodes = elem_nodes.to(torch.int32).contiguous()
        self.x0 = x0.to(torch.float64).contiguous()
        self.rho0 = rho0.to(torch.float64).contiguous()
        self.n_elem = int(self.elem_nodes.shape[0])
        self.n_nodes = int(self.x0.shape[1])
        self._desc = _MeshDesc(dim, k, nq, self.n_elem, self.n_nodes, _ptr(self.elem_nodes),
                               _ptr(self.x0), _ptr(self.rho0))
        nbytes = L.hydro_ctx_workspace_bytes(ctypes.byref(self._desc))
        if nbytes == 0:
            raise HydroError(HYDRO_ERR_ARG, "hydro_ctx_workspace_bytes")
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.x0.device)
        base = self.workspace.data_ptr()
        aligned = (base + 255) & ~255
        self._ws_ptr = ctypes.c_void_p(aligned)
        self._ws_bytes = nbytes
        h = ctypes.c_void_p()
        _check(L.hydro_ctx_create(ctypes.byref(self._desc), self._ws_ptr, nbytes, _stream(stream),
                                  ctypes.byref(h)), "hydro_ctx_create")
        self._h = h
        self.ne = k ** dim
        self.nd = (k + 1) ** dim

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            if getattr(self, "_h", None) and self._h.value:
                lib().hydro_ctx_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def mq(self) -> torch.Tensor:
        """View of the per-quadrature-point mass m_q inside the workspace ([E][nq^dim])."""
        nq = self.nq ** self.dim
        off = 256 * ((8 * 128 + 255) // 256) + 256 * ((32 + 255) // 256)
        start = self._ws_ptr.value - self.workspace.data_ptr() + off
        return self.workspace[start:start + 8 * self.n_elem * nq].view(torch.float64).view(self.n_elem, nq)

    def force_full(self, x, v, e, gamma, visc: Visc, cfl: Cfl, w=None, F1=None, FTw=None,
                   dt=None, stream=None):
        if F1 is None:
            F1 = torch.empty((self.dim, self.n_nodes), dtype=torch.float64, device=x.device)
        if FTw is None:
            FTw = torch.empty((self.n_elem, self.ne), dtype=torch.float64, device=x.device)
        if dt is None:
            dt = torch.empty(1, dtype=torch.float64, device=x.device)
        _check(lib().hydro_force_full(self._h, _ptr(x), _ptr(v), _ptr(e), _ptr(w), _ptr(gamma),
                                      visc.c(), cfl.c(), _ptr(F1), _ptr(FTw), _ptr(dt),
                                      _stream(stream)), "hydro_force_full")
        return F1, FTw, dt

    def force_full_store(self, x, v, e, gamma, visc: Visc, cfl: Cfl, F1=None, FTw=None, dt=None,
                         S=None, stream=None):
        """hydro_force_full (w = v) that also stores S_q; returns (F1, FTw, dt, S)."""
        dev = x.device
        if F1 is None:
            F1 = torch.empty((self.dim, self.n_nodes), dtype=torch.float64, device=dev)
        if FTw is None:
            FTw = torch.empty((self.n_elem, self.ne), dtype=torch.float64, device=dev)
        if dt is None:
            dt = torch.empty(1, dtype=torch.float64, device=dev)
        if S is None:
            S = torch.empty(lib().hydro_force_stress_bytes(self._h) // 8, dtype=torch.float64, device=dev)
        _check(lib().hydro_force_full_store(self._h, _ptr(x), _ptr(v), _ptr(e), _ptr(gamma), visc.c(),
                                            cfl.c(), _ptr(F1), _ptr(FTw), _ptr(dt), _ptr(S),
                                            _stream(stream)), "hydro_force_full_store")
        return F1, FTw, dt, S

    def force_transpose(self, S, w, FTw=None, stream=None):
        if FTw is None:
            FTw = torch.empty((self.n_elem, self.ne), dtype=torch.float64, device=w.device)
        _check(lib().hydro_force_transpose(self._h, _ptr(S), _ptr(w), _ptr(FTw), _stream(stream)),
               "hydro_force_transpose")
        return FTw

    def dt_estimate(self, x, v, e, gamma, visc: Visc, cfl: Cfl, dt=None, stream=None):
        if dt is None:
            dt = torch.empty(1, dtype=torch.float64, device=x.device)
        _check(lib().hydro_dt_estimate(self._h, _ptr(x), _ptr(v), _ptr(e), _ptr(gamma), visc.c(),
                                       cfl.c(), _ptr(dt), _stream(stream)), "hydro_dt_estimate")
        return dt

    def status_sync(self, stream=None):
        """Returns (status_code, first_bad_element) and clears the sticky status."""
        fb = ctypes.c_int64(-1)
        rc = lib().hydro_status_sync(self._h, _stream(stream), ctypes.byref(fb))
        if rc in (HYDRO_ERR_ARG, HYDRO_ERR_CUDA):
            raise HydroError(rc, "hydro_status_sync")
        return rc, fb.value


class SamplePlan:
    """hydro_sample_create: closure of a sample element set, batched over B instances."""

    def __init__(self, ctx: HydroContext, sample_elems, B: int):
        import numpy as np
        L = lib()
        s = np.ascontiguousarray(np.asarray(sample_elems, dtype=np.int32))
        h = ctypes.c_void_p()
        _check(L.hydro_sample_create(ctx.handle, s.ctypes.data_as(ctypes.c_void_p), s.size, B,
                                     ctypes.byref(h)), "hydro_sample_create")
        self._h, self.ctx, self.B = h, ctx, B
        v = [ctypes.c_int64() for _ in range(5)]
        _check(L.hydro_sample_info(h, *[ctypes.byref(t) for t in v]), "hydro_sample_info")
        self.n_cl, self.n_cl_nodes, self.n_s0_nodes, self.s_v, self.s_e = [t.value for t in v]
        self.closure_elems = np.zeros(self.n_cl, dtype=np.int32)
        self.closure_nodes = np.zeros(self.n_cl_nodes, dtype=np.int64)
        self.s0_nodes = np.zeros(self.n_s0_nodes, dtype=np.int64)
        _check(L.hydro_sample_lists(h, self.closure_elems.ctypes.data_as(ctypes.c_void_p),
                                    self.closure_nodes.ctypes.data_as(ctypes.c_void_p),
                                    self.s0_nodes.ctypes.data_as(ctypes.c_void_p)), "hydro_sample_lists")

    def __del__(self):
        try:
            if getattr(self, "_h", None) and self._h.value:
                lib().hydro_sample_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def force_sampled(self, x_S, v_S, e_S, gamma, visc: Visc, cfl: Cfl, w_S=None, F1_rows=None,
                      FTw_rows=None, dt=None, stream=None):
        dev = x_S.device
        if F1_rows is None:
            F1_rows = torch.empty((self.s_v, self.B), dtype=torch.float64, device=dev)
        if FTw_rows is None:
            FTw_rows = torch.empty((self.s_e, self.B), dtype=torch.float64, device=dev)
        if dt is None:
            dt = torch.empty(self.B, dtype=torch.float64, device=dev)
        _check(lib().hydro_force_sampled(self._h, _ptr(x_S), _ptr(v_S), _ptr(e_S), _ptr(w_S),
                                         _ptr(gamma), visc.c(), cfl.c(), _ptr(F1_rows),
                                         _ptr(FTw_rows), _ptr(dt), _stream(stream)),
               "hydro_force_sampled")
        return F1_rows, FTw_rows, dt

    def status_sync(self, stream=None):
        fb = ctypes.c_int64(-1)
        rc = lib().hydro_sample_status_sync(self._h, _stream(stream), ctypes.byref(fb))
        if rc in (HYDRO_ERR_ARG, HYDRO_ERR_CUDA):
            raise HydroError(rc, "hydro_sample_status_sync")
        return rc, fb.value


def rom_lift(Phi: torch.Tensor, os_: torch.Tensor, Y: torch.Tensor, out: Optional[torch.Tensor] = None,
             stream=None) -> torch.Tensor:
    """out[r][b] = os[r] (1-D) or os[r][b] (2-D) + sum_k Phi[r][k] Y[k][b]."""
    rows, n = Phi.shape
    B = Y.shape[1]
    if out is None:
        out = torch.empty((rows, B), dtype=torch.float64, device=Phi.device)
    _check(lib().hydro_rom_lift(rows, n, B, _ptr(Phi), _ptr(os_), 1 if os_.dim() == 2 else 0,
                                _ptr(Y), _ptr(out), _stream(stream)), "hydro_rom_lift")
    return out


def rom_window_transition(T: torch.Tensor, c: torch.Tensor, Y: torch.Tensor,
                          out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Initial reduced coordinates of time window w, PAPER Eq. ic-tw / ic2-tw
    (P:1223-1264): Y_w = T Y_{w-1} + c with the offline T [n_w][n_{w-1}] and c ([n_w] or
    [n_w][B]) -- the lift primitive (hydro_rom_lift) on reduced dimensions."""
    return rom_lift(T, c, Y, out=out, stream=stream)


def index_copy_add(n: int, dim: int, src: torch.Tensor, ld_src: int, src_idx, dst: torch.Tensor,
                   ld_dst: int, dst_idx, add: bool, stream=None):
    """dst[c, dst_idx[i]] (+)= src[c, src_idx[i]] over [dim][ld] row blocks -- hydro_index_copy_add.
    Index tensors: device int64 or None (identity)."""
    _check(lib().hydro_index_copy_add(n, dim, _ptr(src), ld_src, _ptr(src_idx), _ptr(dst), ld_dst,
                                      _ptr(dst_idx), 1 if add else 0, _stream(stream)), "hydro_index_copy_add")


def window_ops(Phi_new: torch.Tensor, Phi_old: torch.Tensor, os_new: torch.Tensor,
               os_old: torch.Tensor, fom: Optional["Fom"] = None, field: int = 0, stream=None):
    """(T, c) of the time-window transition (hydro_window_ops): Eq. ic-tw when fom is None or
    field == 0, the M-oblique Eq. ic2-tw with M_V (field 1) or M_E (field 2) otherwise.
    Offsets [N] or [N][B]; returns device T [n_new][n_old], c [n_new][B]."""
    N, n_new = Phi_new.shape
    n_old = Phi_old.shape[1]
    osn = (os_new if os_new.dim() == 2 else os_new.reshape(N, 1)).contiguous()
    oso = (os_old if os_old.dim() == 2 else os_old.reshape(N, 1)).contiguous()
    B = osn.shape[1]
    T = torch.empty((n_new, n_old), dtype=torch.float64, device=Phi_new.device)
    c = torch.empty((n_new, B), dtype=torch.float64, device=Phi_new.device)
    Pn, Po = Phi_new.contiguous(), Phi_old.contiguous()
    _check(lib().hydro_window_ops(fom._h if fom is not None else None, field, N, n_new, n_old, B, _ptr(Pn),
                                  _ptr(Po), _ptr(osn), _ptr(oso), _ptr(T), _ptr(c), _stream(stream)),
           "hydro_window_ops")
    return T, c


def gappy_pinv(U: torch.Tensor, rows, stream=None) -> torch.Tensor:
    """P = (U[rows, :])^+ [m][s] (device) -- hydro_gappy_pinv, the offline factor of the
    hyper-reduced projection.  U device [N][m]; rows: host int64 [s]."""
    import numpy as _np
    N, m = U.shape
    r = _np.ascontiguousarray(_np.asarray(rows, dtype=_np.int64))
    P = torch.empty((m, r.size), dtype=torch.float64, device=U.device)
    _check(lib().hydro_gappy_pinv(_ptr(U.contiguous()), N, m,
                                  r.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), r.size, _ptr(P),
                                  _stream(stream)), "hydro_gappy_pinv")
    return P


def offline_projectors(Phi_x: torch.Tensor, Phi_v: torch.Tensor, Phi_e: torch.Tensor,
                       v_os: torch.Tensor, rows_v, rows_e, stream=None):
    """Offline operators of the hyper-reduced online step over the sample-mesh rows (SURVEY
    R21), all on the GPU: P_v = (Z_v^T Phi_v)^+ [nv][s_v], P_e = (Z_e^T Phi_e)^+ [ne][s_e]
    (Eq. sol-ls-hyper, SNS with M = I P:985-1000; hydro_gappy_pinv), and
    C_xv = Phi_x^T Phi_v [nx][nv], c_x = Phi_x^T v_os [nx] (hydro_window_ops with
    os_new = 0, os_old = v_os).  rows_v / rows_e: host indices of the sampled rows among the
    basis rows, in the order of hydro_force_sampled's F1_rows / FTw_rows."""
    P_v = gappy_pinv(Phi_v, rows_v, stream)
    P_e = gappy_pinv(Phi_e, rows_e, stream)
    zero = torch.zeros_like(v_os)
    C_xv, c_x = window_ops(Phi_x, Phi_v, zero, v_os, stream=stream)
    return P_v, P_e, C_xv, c_x.reshape(-1).contiguous()


def rom_window_offset(Phi_prev: torch.Tensor, os_prev: torch.Tensor, Y_prev: torch.Tensor,
                      n_new: int = 0, stream=None):
    """Eq. previous_os: os_w = os_{w-1} + Phi_{w-1} Y_{w-1} ([rows][B]) and the new
    window's zero initial coordinates ([n_new][B]) -- hydro_rom_window_offset."""
    rows, n = Phi_prev.shape
    B = Y_prev.shape[1]
    os_new = torch.empty((rows, B), dtype=torch.float64, device=Phi_prev.device)
    Y_new = torch.empty((n_new, B), dtype=torch.float64, device=Phi_prev.device) if n_new > 0 else None
    _check(lib().hydro_rom_window_offset(rows, n, B, _ptr(Phi_prev), _ptr(os_prev), 1 if os_prev.dim() == 2 else 0,
                                         _ptr(Y_prev.contiguous()), _ptr(os_new), n_new, _ptr(Y_new),
                                         _stream(stream)), "hydro_rom_window_offset")
    return os_new, Y_new


def basis_tproduct(Phi: torch.Tensor, X: torch.Tensor, stream=None) -> torch.Tensor:
    """Phi^T X ([n][B], device) -- hydro_basis_tproduct (deterministic split-K)."""
    N, n = Phi.shape
    X2 = X.reshape(N, -1).contiguous()
    out = torch.empty((n, X2.shape[1]), dtype=torch.float64, device=Phi.device)
    _check(lib().hydro_basis_tproduct(N, n, X2.shape[1], _ptr(Phi.contiguous()), _ptr(X2), _ptr(out),
                                      _stream(stream)), "hydro_basis_tproduct")
    return out


def rom_previous_window(Phi_prev, os_prev, Y_prev, Phi_new, Phi_x_new, stream=None):
    """The previous-window offsets of one transition for all three fields:
    Phi_prev / os_prev / Y_prev / Phi_new: (x, v, e) tuples of the old window's bases, offsets and
    final coordinates and the new window's bases.  Returns (x_os, v_os, e_os) [rows][B], the new
    window's zero coordinates (Yx, Yv, Ye) and its per-instance c_x = Phi_x,w^T v_os,w [nx][B]."""
    outs, Ys = [], []
    for P0, o0, Y0, P1 in zip(Phi_prev, os_prev, Y_prev, Phi_new):
        o1, Y1 = rom_window_offset(P0, o0, Y0, n_new=P1.shape[1], stream=stream)
        outs.append(o1)
        Ys.append(Y1)
    c_x = basis_tproduct(Phi_x_new, outs[1], stream=stream)
    return tuple(outs), tuple(Ys), c_x


def rom_windowed_advance(windows, Yx, Yv, Ye, gamma, visc: Visc, cfl: Cfl, t0: float, dt,
                         ctrl: DtCtrl = DtCtrl(), max_iters=1000000, stream=None):
    """The time-windowing online phase: for each window advance with its own
    RomStepper to its end time (hydro_rom_advance), then map the reduced coordinates into
    the next window's bases (rom_window_transition).  windows: list of dicts with keys
    stepper, t_end and, except for the last, trans = ((Tx, cx), (Tv, cv), (Te, ce)) as
    device tensors.  Returns (Yx, Yv, Ye, t[B], next_dt[B], per-window (accepted, rejected));
    the returned coordinates are new tensors where a transition changed their dimension."""
    t, h, stats, tB = t0, list(dt), [], None
    for w in windows:
        tB, h, ns, nr, _ = w["stepper"].advance(Yx, Yv, Ye, gamma, visc, cfl, t, w["t_end"], h,
                                                ctrl, max_iters, stream)
        stats.append((ns, nr))
        t = w["t_end"]
        if w.get("trans") is not None:
            (Tx, cx), (Tv, cv), (Te, ce) = w["trans"]
            Yx = rom_window_transition(Tx, cx, Yx, stream=stream)
            Yv = rom_window_transition(Tv, cv, Yv, stream=stream)
            Ye = rom_window_transition(Te, ce, Ye, stream=stream)
    return Yx, Yv, Ye, tB, h, stats


def rom_windowed_advance_previous(plan, windows, x_os, v_os, e_os, c_x, Yx, Yv, Ye, gamma,
                                  visc: Visc, cfl: Cfl, t0: float, dt, ctrl: DtCtrl = DtCtrl(),
                                  max_iters=1000000, stream=None):
    """Time windows with previous-window offsets: window 1 runs with the given
    offsets and c_x; at each transition the offsets of window w are the lifts of window w-1's
    final state (rom_previous_window: hydro_rom_window_offset per field, c_x by
    hydro_basis_tproduct), the coordinates restart at 0, and a new RomStepper is made with
    the window's bases and operators.  windows: list of dicts with keys Phi_x, Phi_v, Phi_e,
    R_v, R_e, C_xv (device) and t_end.  Returns (Yx, Yv, Ye, t[B], next_dt[B], per-window
    (accepted, rejected), per-transition milliseconds (CUDA events))."""
    t, h, stats, tB, trans_ms = t0, list(dt), [], None, []
    os_ = (x_os, v_os, e_os)
    cx = c_x
    for wi, w in enumerate(windows):
        st = RomStepper(plan, w["Phi_x"], w["Phi_v"], w["Phi_e"], *os_, w["R_v"], w["R_e"], w["C_xv"], cx)
        tB, h, ns, nr, _ = st.advance(Yx, Yv, Ye, gamma, visc, cfl, t, w["t_end"], h, ctrl, max_iters, stream)
        stats.append((ns, nr))
        t = w["t_end"]
        if wi + 1 < len(windows):
            nw = windows[wi + 1]
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            os_, (Yx, Yv, Ye), cx = rom_previous_window(
                (w["Phi_x"], w["Phi_v"], w["Phi_e"]), os_, (Yx, Yv, Ye),
                (nw["Phi_x"], nw["Phi_v"], nw["Phi_e"]), nw["Phi_x"], stream=stream)
            b.record()
            torch.cuda.synchronize()
            trans_ms.append(a.elapsed_time(b))
    return Yx, Yv, Ye, tB, h, stats, trans_ms


def pod(S: torch.Tensor, eps: float = 0.9999, max_k: Optional[int] = None, stream=None):
    """POD basis of the snapshots S (device [ns][N], one snapshot per row): (Phi [N][k],
    sigma [ns] numpy) -- hydro_pod (energy criterion of P:955-963)."""
    import numpy as _np
    ns, N = S.shape
    max_k = min(ns, 128) if max_k is None else max_k
    S = S.contiguous()
    Phi = torch.empty((N, max_k), dtype=torch.float64, device=S.device)
    sig = (ctypes.c_double * ns)()
    k = ctypes.c_int(0)
    _check(lib().hydro_pod(_ptr(S), ns, N, eps, max_k, _ptr(Phi), sig, ctypes.byref(k),
                           _stream(stream)), "hydro_pod")
    return Phi[:, :k.value].contiguous(), _np.array(sig[:])


def deim(U: torch.Tensor, stream=None):
    """Greedy DEIM indices (numpy int64 [m]) of the basis U (device [N][m]) -- hydro_deim."""
    import numpy as _np
    N, m = U.shape
    idx = (ctypes.c_int64 * m)()
    _check(lib().hydro_deim(_ptr(U.contiguous()), N, m, idx, _stream(stream)), "hydro_deim")
    return _np.array(idx[:], dtype=_np.int64)


def qdeim(U: torch.Tensor, stream=None):
    """Q-DEIM indices (numpy int64 [m]) of the basis U (device [N][m]) -- hydro_qdeim."""
    import numpy as _np
    N, m = U.shape
    idx = (ctypes.c_int64 * m)()
    _check(lib().hydro_qdeim(_ptr(U.contiguous()), N, m, idx, _stream(stream)), "hydro_qdeim")
    return _np.array(idx[:], dtype=_np.int64)


def deim_oversampled(U: torch.Tensor, n_s: int, stream=None):
    """Oversampled greedy DEIM indices (numpy int64 [n_s]) -- hydro_deim_oversampled."""
    import numpy as _np
    N, m = U.shape
    idx = (ctypes.c_int64 * n_s)()
    _check(lib().hydro_deim_oversampled(_ptr(U.contiguous()), N, m, n_s, idx, _stream(stream)),
           "hydro_deim_oversampled")
    return _np.array(idx[:], dtype=_np.int64)


def rom_project_workspace(n: int, s_rows: int, B: int, device="cuda") -> torch.Tensor:
    nb = lib().hydro_rom_project_workspace_bytes(n, s_rows, B)
    return torch.empty(max(nb, 8), dtype=torch.uint8, device=device)


def rom_project(P: torch.Tensor, f: torch.Tensor, out: Optional[torch.Tensor] = None,
                workspace: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """r[i][b] = sum_s P[i][s] f[s][b] (deterministic split-K)."""
    n, s_rows = P.shape
    B = f.shape[1]
    if out is None:
        out = torch.empty((n, B), dtype=torch.float64, device=P.device)
    if workspace is None:
        workspace = rom_project_workspace(n, s_rows, B, P.device)
    _check(lib().hydro_rom_project(n, s_rows, B, _ptr(P), _ptr(f), _ptr(out), _ptr(workspace),
                                   workspace.numel(), _stream(stream)), "hydro_rom_project")
    return out


class Fom:
    """Full-order RK2-average stepper (hydro_fom_*; PAPER Eq. RK2-avg) on a context.
    bc_dofs: constrained velocity dofs (flat c*n_nodes + node) of v.n = 0."""

    def __init__(self, ctx: HydroContext, bc_dofs, stream=None):
        import numpy as np
        L = lib()
        bc = np.ascontiguousarray(np.asarray(bc_dofs, dtype=np.int64))
        h = ctypes.c_void_p()
        _check(L.hydro_fom_create(ctx.handle, bc.ctypes.data_as(ctypes.c_void_p) if bc.size else None,
                                  bc.size, _stream(stream), ctypes.byref(h)), "hydro_fom_create")
        self._h, self.ctx = h, ctx

    def __del__(self):
        try:
            if getattr(self, "_h", None) and self._h.value:
                lib().hydro_fom_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def mass_v(self, v, out=None, stream=None):
        out = torch.empty_like(v) if out is None else out
        _check(lib().hydro_mass_v_apply(self._h, _ptr(v), _ptr(out), _stream(stream)), "hydro_mass_v_apply")
        return out

    def solve_v(self, rhs, tol=1e-12, max_iter=500, out=None, stream=None):
        out = torch.empty_like(rhs) if out is None else out
        it, rel = ctypes.c_int(0), ctypes.c_double(0.0)
        _check(lib().hydro_mass_v_solve(self._h, _ptr(rhs), _ptr(out), tol, max_iter, ctypes.byref(it),
                                        ctypes.byref(rel), _stream(stream)), "hydro_mass_v_solve")
        return out, it.value, rel.value

    def mass_e(self, e, out=None, stream=None):
        out = torch.empty_like(e) if out is None else out
        _check(lib().hydro_mass_e_apply(self._h, _ptr(e), _ptr(out), _stream(stream)), "hydro_mass_e_apply")
        return out

    def indicator(self, x, v, e, gamma, visc: Visc, cfl: Cfl, Phi_v, Phi_e, U1, Z1, U2, Z2, stream=None):
        """Theorem-2 integrands (eta_v, eta_e) at the state (x, v, e) -- hydro_rom_indicator."""
        Z1 = [int(i) for i in Z1]
        Z2 = [int(i) for i in Z2]
        z1, z2 = (ctypes.c_int64 * len(Z1))(*Z1), (ctypes.c_int64 * len(Z2))(*Z2)
        eta = (ctypes.c_double * 2)()
        ops = [t.contiguous() for t in (Phi_v, Phi_e, U1, U2)]
        _check(lib().hydro_rom_indicator(self._h, _ptr(x), _ptr(v), _ptr(e), _ptr(gamma), visc.c(), cfl.c(),
                                         ops[0].shape[1], _ptr(ops[0]), ops[1].shape[1], _ptr(ops[1]),
                                         ops[2].shape[1], _ptr(ops[2]), len(Z1), z1, ops[3].shape[1],
                                         _ptr(ops[3]), len(Z2), z2, eta, _stream(stream)),
               "hydro_rom_indicator")
        return eta[0], eta[1]

    def solve_e(self, rhs, out=None, stream=None):
        out = torch.empty_like(rhs) if out is None else out
        _check(lib().hydro_mass_e_solve(self._h, _ptr(rhs), _ptr(out), _stream(stream)), "hydro_mass_e_solve")
        return out

    def energy(self, v, e, stream=None):
        k, i = ctypes.c_double(0.0), ctypes.c_double(0.0)
        _check(lib().hydro_fom_energy(self._h, _ptr(v), _ptr(e), ctypes.byref(k), ctypes.byref(i),
                                      _stream(stream)), "hydro_fom_energy")
        return k.value, i.value

    def step(self, x, v, e, gamma, visc: Visc, cfl: Cfl, dt: float, cg_tol=1e-12, cg_max_iter=500,
             stream=None):
        """In-place RK2-average step; returns (dt_estimate, cg_iterations)."""
        d, it = ctypes.c_double(0.0), ctypes.c_int(0)
        _check(lib().hydro_rk2avg_step(self._h, _ptr(x), _ptr(v), _ptr(e), _ptr(gamma), visc.c(), cfl.c(),
                                       dt, cg_tol, cg_max_iter, ctypes.byref(d), ctypes.byref(it),
                                       _stream(stream)), "hydro_rk2avg_step")
        return d.value, it.value

    def stage_state(self, x_half=None, v_half=None, e_half=None, stream=None):
        """Copy the last step's half-stage state (x, v, e)^{n+1/2} into the given tensors."""
        _check(lib().hydro_fom_stage_state(self._h, _ptr(x_half), _ptr(v_half), _ptr(e_half),
                                           _stream(stream)), "hydro_fom_stage_state")

    def advance(self, x, v, e, gamma, visc: Visc, cfl: Cfl, t0: float, t_final: float, dt: float,
                ctrl: DtCtrl = DtCtrl(), max_steps=1000000, cg_tol=1e-12, cg_max_iter=500,
                stream=None):
        """In-place time loop t0 -> t_final under the controller of P:549-566.
        Returns (t_reached, next_dt, accepted_steps, rejected_steps)."""
        h, t = ctypes.c_double(dt), ctypes.c_double(0.0)
        ns, nr = ctypes.c_int(0), ctypes.c_int(0)
        _check(lib().hydro_fom_advance(self._h, _ptr(x), _ptr(v), _ptr(e), _ptr(gamma), visc.c(),
                                       cfl.c(), ctrl.c(), t0, t_final, ctypes.byref(h), max_steps,
                                       cg_tol, cg_max_iter, ctypes.byref(t), ctypes.byref(ns),
                                       ctypes.byref(nr), _stream(stream)), "hydro_fom_advance")
        return t.value, h.value, ns.value, nr.value


class RomStepper:
    """Hyper-reduced RK2-average online step (hydro_rom_*; PAPER Eq. RK2-avg-rom-hr
    P:847-906) for the B instances of a SamplePlan.  Keeps references to its operands."""

    def __init__(self, plan: SamplePlan, Phi_x, Phi_v, Phi_e, x_os, v_os, e_os, R_v, R_e, C_xv, c_x):
        self._keep = [t.contiguous() for t in (Phi_x, Phi_v, Phi_e, x_os, v_os, e_os, R_v, R_e, C_xv, c_x)]
        Phi_x, Phi_v, Phi_e, x_os, v_os, e_os, R_v, R_e, C_xv, c_x = self._keep
        flags = ((1 if x_os.dim() == 2 else 0) | (2 if v_os.dim() == 2 else 0) | (4 if e_os.dim() == 2 else 0)
                 | (8 if c_x.dim() == 2 else 0))
        h = ctypes.c_void_p()
        _check(lib().hydro_rom_create(plan._h, Phi_x.shape[1], Phi_v.shape[1], Phi_e.shape[1], _ptr(Phi_x),
                                      _ptr(Phi_v), _ptr(Phi_e), _ptr(x_os), _ptr(v_os), _ptr(e_os), flags,
                                      _ptr(R_v), _ptr(R_e), _ptr(C_xv), _ptr(c_x), ctypes.byref(h)),
               "hydro_rom_create")
        self._h, self.plan = h, plan

    def __del__(self):
        try:
            if getattr(self, "_h", None) and self._h.value:
                lib().hydro_rom_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def step(self, Yx, Yv, Ye, gamma, visc: Visc, cfl: Cfl, dt, dt_est=None, stream=None):
        """In place on (Yx, Yv, Ye); dt: device [B]; returns dt_est (device [B])."""
        if dt_est is None:
            dt_est = torch.empty_like(dt)
        _check(lib().hydro_rom_rk2avg_step(self._h, _ptr(Yx), _ptr(Yv), _ptr(Ye), _ptr(gamma), visc.c(),
                                           cfl.c(), _ptr(dt), _ptr(dt_est), _stream(stream)),
               "hydro_rom_rk2avg_step")
        return dt_est

    def advance(self, Yx, Yv, Ye, gamma, visc: Visc, cfl: Cfl, t0: float, t_final: float, dt,
                ctrl: DtCtrl = DtCtrl(), max_iters=1000000, stream=None):
        """In-place online time loop t0 -> t_final for every instance under the controller
        of P:549-566.  dt: host sequence [B] of first trial steps.  Returns (t [B], next dt [B],
        accepted [B], rejected [B], batched steps run) as numpy arrays / int."""
        import numpy as _np
        B = self.plan.B
        h = (ctypes.c_double * B)(*[float(d) for d in dt])
        t = (ctypes.c_double * B)()
        ns, nr = (ctypes.c_int * B)(), (ctypes.c_int * B)()
        it = ctypes.c_int(0)
        _check(lib().hydro_rom_advance(self._h, _ptr(Yx), _ptr(Yv), _ptr(Ye), _ptr(gamma), visc.c(),
                                       cfl.c(), ctrl.c(), t0, t_final, h, max_iters, t, ns, nr,
                                       ctypes.byref(it), _stream(stream)), "hydro_rom_advance")
        return (_np.array(t[:]), _np.array(h[:]), _np.array(ns[:]), _np.array(nr[:]), it.value)
