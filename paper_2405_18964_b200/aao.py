"""Thin Python binding of the C-ABI library libaao.so (include/aao.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  PyTorch provides device memory and streams.  There is no CPU
fallback: if libaao.so is missing or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AAO_LIB", os.path.join(_HERE, "libaao.so"))
_lib = None

AAO_STOKES, AAO_OSEEN = 0, 1
STATUS = {0: "AAO_OK", 1: "AAO_NOT_CONVERGED", -1: "AAO_ERR_CONFIG", -2: "AAO_ERR_SHAPE",
          -3: "AAO_ERR_CUDA", -4: "AAO_ERR_OOM", -5: "AAO_ERR_NUMERIC"}


class Config(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("n_cells", ctypes.c_int), ("x_lo", ctypes.c_double),
                ("x_hi", ctypes.c_double), ("n_t", ctypes.c_int), ("T", ctypes.c_double),
                ("beta", ctypes.c_double), ("nu", ctypes.c_double), ("problem", ctypes.c_int),
                ("wind_q2", ctypes.POINTER(ctypes.c_double)), ("mg_cycles", ctypes.c_int),
                ("pre_sweeps", ctypes.c_int), ("post_sweeps", ctypes.c_int), ("omega", ctypes.c_double),
                ("cheb_iters", ctypes.c_int), ("uzawa_iters", ctypes.c_int), ("uzawa_mu", ctypes.c_double),
                ("pmode", ctypes.c_int), ("inner_eps", ctypes.c_double), ("inner_maxit", ctypes.c_int),
                ("freq_chunk", ctypes.c_int)]


class Krylov(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("restart", ctypes.c_int), ("max_iters", ctypes.c_int),
                ("store_z", ctypes.c_int)]


class Info(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("restarts", ctypes.c_int), ("converged", ctypes.c_int),
                ("breakdown", ctypes.c_int), ("final_relres", ctypes.c_double),
                ("true_relres", ctypes.c_double), ("precond_applies", ctypes.c_int),
                ("ms_total", ctypes.c_double), ("inner_its_total", ctypes.c_long), ("inner_its_max", ctypes.c_int),
                ("ms_precond", ctypes.c_double), ("ms_kkt", ctypes.c_double), ("ms_orth", ctypes.c_double),
                ("store_z", ctypes.c_int)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


EXPORTS = ["aao_config_defaults", "aao_create", "aao_destroy", "aao_last_error", "aao_vector_len",
           "aao_device_bytes", "aao_pack", "aao_unpack", "aao_build_rhs", "aao_build_rhs_general", "aao_arnoldi", "aao_kkt_apply",
           "aao_precond_apply",
           "aao_gmres_solve", "aao_gmres_solve_host", "aao_debug_freq_block", "aao_set_timing",
           "aao_last_phase_ms", "aao_last_launch_count", "aao_profile_smoother", "aao_profile_read",
           "aao_last_inner_iterations"]


def load(path: str = LIB_PATH):
    """Load libaao.so and declare the C signatures (raises if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(path)
    vp, dp, i, st = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_int
    L.aao_config_defaults.argtypes = [ctypes.POINTER(Config)]
    L.aao_config_defaults.restype = None
    L.aao_create.argtypes = [ctypes.POINTER(Config), ctypes.POINTER(vp)]
    L.aao_create.restype = st
    L.aao_destroy.argtypes = [vp]
    L.aao_destroy.restype = None
    L.aao_last_error.argtypes = [vp]
    L.aao_last_error.restype = ctypes.c_char_p
    L.aao_vector_len.argtypes = [vp]
    L.aao_vector_len.restype = ctypes.c_size_t
    L.aao_device_bytes.argtypes = [vp]
    L.aao_device_bytes.restype = ctypes.c_size_t
    for name in ("aao_pack", "aao_unpack", "aao_build_rhs", "aao_kkt_apply", "aao_precond_apply"):
        getattr(L, name).argtypes = [vp, vp, vp, vp]
        getattr(L, name).restype = st
    L.aao_arnoldi.argtypes = [vp, vp, i, dp, ctypes.POINTER(ctypes.c_int), vp]
    L.aao_arnoldi.restype = st
    L.aao_build_rhs_general.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.aao_build_rhs_general.restype = st
    L.aao_gmres_solve.argtypes = [vp, vp, vp, ctypes.POINTER(Krylov), ctypes.POINTER(Info), dp, i, vp]
    L.aao_gmres_solve.restype = st
    L.aao_gmres_solve_host.argtypes = [vp, dp, dp, ctypes.POINTER(Krylov), ctypes.POINTER(Info), dp, i, vp]
    L.aao_gmres_solve_host.restype = st
    L.aao_debug_freq_block.argtypes = [vp, i, dp, vp]
    L.aao_debug_freq_block.restype = st
    L.aao_set_timing.argtypes = [vp, i]
    L.aao_set_timing.restype = st
    L.aao_last_phase_ms.argtypes = [vp, dp]
    L.aao_last_phase_ms.restype = st
    L.aao_profile_smoother.argtypes = [vp, i]
    L.aao_profile_smoother.restype = st
    L.aao_profile_read.argtypes = [vp, dp]
    L.aao_profile_read.restype = st
    L.aao_last_inner_iterations.argtypes = [vp, ctypes.POINTER(ctypes.c_int), i]
    L.aao_last_inner_iterations.restype = ctypes.c_int
    L.aao_last_launch_count.argtypes = [vp]
    L.aao_last_launch_count.restype = ctypes.c_long
    _lib = L
    return L


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


class AAOError(RuntimeError):
    pass


class Context:
    """One assembled problem on the current CUDA device (wraps aao_ctx*)."""

    def __init__(self, dim, n_cells, x_lo, x_hi, n_t, T, beta, nu, problem="stokes", wind_q2=None,
                 mg_cycles=4, pre_sweeps=2, post_sweeps=2, omega=1.0, cheb_iters=10, uzawa_iters=6,
                 uzawa_mu=0.75, nonlinear=False, inner_eps=1e-2, inner_maxit=60, freq_chunk=0):
        import torch
        if not torch.cuda.is_available():
            raise AAOError("no CUDA device: the aao hot path has no CPU fallback")
        self.torch = torch
        L = load()
        cfg = Config()
        L.aao_config_defaults(ctypes.byref(cfg))
        cfg.dim, cfg.n_cells, cfg.x_lo, cfg.x_hi = dim, n_cells, x_lo, x_hi
        cfg.n_t, cfg.T, cfg.beta, cfg.nu = n_t, T, beta, nu
        cfg.problem = AAO_OSEEN if problem == "oseen" else AAO_STOKES
        self._wind = None
        if wind_q2 is not None:
            self._wind = np.ascontiguousarray(wind_q2, dtype=np.float64)
            cfg.wind_q2 = self._wind.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        cfg.mg_cycles, cfg.pre_sweeps, cfg.post_sweeps, cfg.omega = mg_cycles, pre_sweeps, post_sweeps, omega
        cfg.cheb_iters, cfg.uzawa_iters, cfg.uzawa_mu = cheb_iters, uzawa_iters, uzawa_mu
        cfg.pmode, cfg.inner_eps, cfg.inner_maxit = (1 if nonlinear else 0), inner_eps, inner_maxit
        cfg.freq_chunk = freq_chunk
        self.nonlinear = bool(nonlinear)
        h = ctypes.c_void_p()
        rc = L.aao_create(ctypes.byref(cfg), ctypes.byref(h))
        if rc != 0:
            raise AAOError(f"aao_create failed: {STATUS.get(rc, rc)}")
        self.h = h
        self.L = L
        self.dim, self.n_t = dim, n_t
        self.n_b = n_t - 1
        self.n_f = self.n_b // 2 + 1
        self.N = L.aao_vector_len(h)
        self.n_block = self.N // (2 * self.n_b)

    @classmethod
    def from_config(cls, cfg, wind_q2=None, **opts):
        """Build from any object with the fields of synth.Config."""
        return cls(cfg.dim, cfg.n_cells, cfg.x_lo, cfg.x_hi, cfg.n_t, cfg.T, cfg.beta, cfg.nu,
                   cfg.problem, wind_q2, **opts)

    def close(self):
        if getattr(self, "h", None):
            self.L.aao_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ helpers
    def _stream(self, stream=None):
        s = stream if stream is not None else self.torch.cuda.current_stream()
        return ctypes.c_void_p(s.cuda_stream)

    def _check(self, rc, what):
        if rc < 0:
            raise AAOError(f"{what}: {STATUS.get(rc, rc)}: {self.L.aao_last_error(self.h).decode()}")
        return rc

    def _vec(self, t):
        torch = self.torch
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
                and t.numel() == self.N):
            raise AAOError(f"expected a contiguous cuda float64 tensor with {self.N} entries")
        return t

    def empty(self):
        return self.torch.empty(self.N, dtype=self.torch.float64, device="cuda")

    # ------------------------------------------------------------------ ABI calls
    def pack(self, x, out=None, stream=None):
        out = self.empty() if out is None else out
        self._check(self.L.aao_pack(self.h, _ptr(self._vec(x)), _ptr(self._vec(out)), self._stream(stream)), "pack")
        return out

    def unpack(self, x, out=None, stream=None):
        out = self.empty() if out is None else out
        self._check(self.L.aao_unpack(self.h, _ptr(self._vec(x)), _ptr(self._vec(out)), self._stream(stream)),
                    "unpack")
        return out

    def build_rhs(self, vd_q2, out=None, stream=None):
        vd = vd_q2 if isinstance(vd_q2, self.torch.Tensor) else self.torch.as_tensor(np.ascontiguousarray(vd_q2))
        vd = vd.to(device="cuda", dtype=self.torch.float64).contiguous()
        out = self.empty() if out is None else out
        self._check(self.L.aao_build_rhs(self.h, _ptr(vd), _ptr(self._vec(out)), self._stream(stream)), "build_rhs")
        return out

    def build_rhs_general(self, vd=None, f=None, g=None, v0=None, out=None, stream=None):
        """aao_build_rhs_general: time-dependent v_d, f, Dirichlet data g (lifting) and v0 (numpy or torch;
        vd, f: (n_b, d, n_s); g: (n_b + 1, d, n_s); v0: (d, n_s))."""
        def dev(a):
            if a is None:
                return None
            t = a if isinstance(a, self.torch.Tensor) else self.torch.as_tensor(np.ascontiguousarray(a))
            return t.to(device="cuda", dtype=self.torch.float64).contiguous()
        arrs = [dev(a) for a in (vd, f, g, v0)]
        out = self.empty() if out is None else out
        ptrs = [_ptr(a) if a is not None else None for a in arrs]
        self._check(self.L.aao_build_rhs_general(self.h, *ptrs, _ptr(self._vec(out)), self._stream(stream)),
                    "build_rhs_general")
        return out

    def arnoldi(self, v0, m, stream=None):
        """aao_arnoldi: m Arnoldi steps on A P^{-1} from v0; returns the unrotated Hessenberg (k+1, k), k = steps
        done (numpy).  Ritz values: np.linalg.eigvals(H[:k, :k])."""
        H = np.zeros((m + 1) * m)
        k = ctypes.c_int(0)
        self._check(self.L.aao_arnoldi(self.h, _ptr(self._vec(v0)), int(m), H.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                       ctypes.byref(k), self._stream(stream)), "arnoldi")
        H = H.reshape(m + 1, m)
        return H[:k.value + 1, :k.value]

    def kkt_apply(self, x, out=None, stream=None):
        out = self.empty() if out is None else out
        self._check(self.L.aao_kkt_apply(self.h, _ptr(self._vec(x)), _ptr(self._vec(out)), self._stream(stream)),
                    "kkt_apply")
        return out

    def precond_apply(self, r, out=None, stream=None):
        out = self.empty() if out is None else out
        self._check(self.L.aao_precond_apply(self.h, _ptr(self._vec(r)), _ptr(self._vec(out)),
                                             self._stream(stream)), "precond_apply")
        return out

    def gmres_solve(self, b, x=None, tol=1e-6, restart=30, max_iters=2000, hist_cap=4096, store_z=False,
                    stream=None):
        x = self.torch.zeros_like(b) if x is None else x
        kry = Krylov(tol, restart, max_iters, 1 if store_z else 0)
        info = Info()
        hist = (ctypes.c_double * hist_cap)()
        rc = self._check(self.L.aao_gmres_solve(self.h, _ptr(self._vec(b)), _ptr(self._vec(x)), ctypes.byref(kry),
                                                ctypes.byref(info), hist, hist_cap, self._stream(stream)),
                         "gmres_solve")
        return x, info.as_dict(), list(hist[:min(info.iterations, hist_cap)]), rc

    def _host_vec(self, a, what):
        """A HOST buffer of N float64: a C-contiguous numpy array or a contiguous CPU torch tensor."""
        torch = self.torch
        if isinstance(a, np.ndarray):
            ok = a.dtype == np.float64 and a.flags["C_CONTIGUOUS"] and a.size == self.N
            if not ok:
                raise AAOError(f"{what}: expected a C-contiguous float64 numpy array with {self.N} entries")
            return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        if isinstance(a, torch.Tensor):
            ok = (a.device.type == "cpu" and a.dtype == torch.float64 and a.is_contiguous() and a.numel() == self.N)
            if not ok:
                raise AAOError(f"{what}: expected a contiguous CPU float64 tensor with {self.N} entries")
            return ctypes.cast(ctypes.c_void_p(a.data_ptr()), ctypes.POINTER(ctypes.c_double))
        raise AAOError(f"{what}: expected a numpy array or a CPU torch tensor")

    def gmres_solve_host(self, b_host, x_host=None, tol=1e-6, restart=30, max_iters=2000, hist_cap=4096,
                         store_z=False, stream=None):
        """End-to-end entry: HOST b and x (numpy float64 or CPU torch float64, pinned or pageable, N entries each);
        the copies are inside the call.  x_host (the initial guess, overwritten by the solution) defaults to zeros."""
        if x_host is None:
            x_host = np.zeros(self.N) if isinstance(b_host, np.ndarray) else self.torch.zeros_like(b_host)
        bp = self._host_vec(b_host, "b_host")
        xp = self._host_vec(x_host, "x_host")
        kry = Krylov(tol, restart, max_iters, 1 if store_z else 0)
        info = Info()
        hist = (ctypes.c_double * hist_cap)()
        rc = self._check(self.L.aao_gmres_solve_host(self.h, bp, xp, ctypes.byref(kry), ctypes.byref(info), hist,
                                                     hist_cap, self._stream(stream)), "gmres_solve_host")
        return x_host, info.as_dict(), list(hist[:min(info.iterations, hist_cap)]), rc

    def debug_freq_block(self, k, stream=None):
        """y_hat_k of the last precond_apply: complex array (2, n_v + n_p)."""
        out = np.zeros(2 * 2 * self.n_block)
        self._check(self.L.aao_debug_freq_block(self.h, k, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                                self._stream(stream)), "debug_freq_block")
        return (out[0::2] + 1j * out[1::2]).reshape(2, self.n_block)

    def phase_ms(self):
        out = (ctypes.c_double * 4)()
        self._check(self.L.aao_last_phase_ms(self.h, out), "phase_ms")
        return list(out)

    def set_timing(self, on=True):
        """aao_set_timing: per-phase device timings (precond phases; GMRES ms_precond / ms_kkt / ms_orth)."""
        self._check(self.L.aao_set_timing(self.h, 1 if on else 0), "set_timing")

    def profile_smoother(self, on=True, reserve=0):
        """Live timing of the velocity-MG launches; `reserve` pre-creates events for that many launches."""
        self._check(self.L.aao_profile_smoother(self.h, (max(2, int(reserve)) if reserve else 1) if on else 0),
                    "profile_smoother")

    def profile_read(self):
        """(ms, algorithmic bytes, launches) of the finest-level SOR sweeps since profile_smoother(True)."""
        out = (ctypes.c_double * 3)()
        self._check(self.L.aao_profile_read(self.h, out), "profile_read")
        return out[0], out[1], int(out[2])

    def last_inner_iterations(self):
        """Nonlinear mode: inner GMRES iterations per stored frequency of the last precond_apply."""
        buf = (ctypes.c_int * self.n_f)()
        n = self._check(self.L.aao_last_inner_iterations(self.h, buf, self.n_f), "last_inner_iterations")
        return list(buf[:n])

    def last_launch_count(self):
        return int(self.L.aao_last_launch_count(self.h))

    def device_bytes(self):
        return int(self.L.aao_device_bytes(self.h))
