"""Thin ctypes binding of the cnpint C ABI (include/cnpint.h).

Argument marshalling only: every step of the AaO matvec, P_α⁻¹ and GMRES runs in the CUDA kernels of
``libcnpint.so`` (built in-tree by ``make`` / ``__graft_entry__.build()``).  PyTorch supplies device
memory (workspace and vectors) and the CUDA stream.  There is no CPU fallback: if the library or a
CUDA device is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# CNPINT_LIB: an alternative in-tree build of the same library (tuning experiments only)
LIB_PATH = os.environ.get("CNPINT_LIB") or os.path.join(_HERE, "libcnpint.so")

STATUS = {0: "CNPINT_OK", -1: "CNPINT_EINVAL", -2: "CNPINT_EUNSUPPORTED", -3: "CNPINT_ECUDA",
          -4: "CNPINT_ESINGULAR", -5: "CNPINT_ENOCONV", -6: "CNPINT_EBREAKDOWN"}
OK, EINVAL, EUNSUPPORTED, ECUDA, ESINGULAR, ENOCONV, EBREAKDOWN = 0, -1, -2, -3, -4, -5, -6

# every symbol include/cnpint.h declares (checked by tests/test_abi.py)
EXPORTS = ["cnpint_workspace_bytes", "cnpint_create", "cnpint_destroy", "cnpint_last_error", "cnpint_set_stream",
           "cnpint_ld", "cnpint_vec_elems", "cnpint_spec_elems", "cnpint_apply_A", "cnpint_apply_P",
           "cnpint_apply_Pinv", "cnpint_time_fft", "cnpint_shifted_solve", "cnpint_time_ifft", "cnpint_gmres",
           "cnpint_apply_Pinv_host", "cnpint_apply_A_host", "cnpint_gmres_host", "cnpint_device_status",
           "cnpint_launch_count", "cnpint_stream_copy", "cnpint_set_debug", "cnpint_profile_enable",
           "cnpint_profile_read", "cnpint_kernel_name", "cnpint_set_time_dependence", "cnpint_gmres_left"]


class CnpintError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Operator(C.Structure):
    _fields_ = [("dim", C.c_int), ("nx", C.c_int), ("ny", C.c_int), ("toeplitz", C.c_int),
                ("sub", C.POINTER(C.c_double)), ("diag", C.POINTER(C.c_double)), ("sup", C.POINTER(C.c_double)),
                ("xs", C.c_double), ("xd", C.c_double), ("xu", C.c_double),
                ("ys", C.c_double), ("yd", C.c_double), ("yu", C.c_double), ("shift", C.c_double)]


class GmresReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("restarts", C.c_int), ("converged", C.c_int),
                ("relres_est", C.c_double), ("relres_true", C.c_double), ("seconds", C.c_double),
                ("history", C.POINTER(C.c_double)), ("history_cap", C.c_int), ("relres_prec", C.c_double)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libcnpint.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OSError(f"{path} not found: build it with `make` (or __graft_entry__.build())")
    lib = C.CDLL(path)
    vp, dp, i64 = C.c_void_p, C.POINTER(C.c_double), C.c_int64
    sig = {
        "cnpint_workspace_bytes": (C.c_size_t, [C.c_int, C.POINTER(Operator), C.c_int]),
        "cnpint_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_double, C.c_double, C.POINTER(Operator),
                                    C.c_int, vp, C.c_size_t, vp]),
        "cnpint_destroy": (None, [vp]),
        "cnpint_last_error": (C.c_char_p, [vp]),
        "cnpint_set_stream": (C.c_int, [vp, vp]),
        "cnpint_ld": (i64, [vp]), "cnpint_vec_elems": (i64, [vp]), "cnpint_spec_elems": (i64, [vp]),
        "cnpint_apply_A": (C.c_int, [vp, vp, vp]), "cnpint_apply_P": (C.c_int, [vp, vp, vp]),
        "cnpint_apply_Pinv": (C.c_int, [vp, vp, vp]),
        "cnpint_time_fft": (C.c_int, [vp, vp, vp]), "cnpint_shifted_solve": (C.c_int, [vp, vp, vp]),
        "cnpint_time_ifft": (C.c_int, [vp, vp, vp]),
        "cnpint_gmres": (C.c_int, [vp, vp, vp, C.c_double, C.c_int, C.c_int, C.POINTER(GmresReport)]),
        "cnpint_gmres_left": (C.c_int, [vp, vp, vp, C.c_double, C.c_int, C.c_int, C.POINTER(GmresReport)]),
        "cnpint_apply_Pinv_host": (C.c_int, [vp, dp, dp]), "cnpint_apply_A_host": (C.c_int, [vp, dp, dp]),
        "cnpint_gmres_host": (C.c_int, [vp, dp, dp, C.c_double, C.c_int, C.c_int, C.POINTER(GmresReport)]),
        "cnpint_device_status": (C.c_int, [vp]), "cnpint_launch_count": (i64, [vp]),
        "cnpint_stream_copy": (C.c_int, [vp, vp, C.c_size_t, vp]), "cnpint_set_debug": (C.c_int, [vp, C.c_int]),
        "cnpint_profile_enable": (C.c_int, [vp, C.c_int]),
        "cnpint_profile_read": (C.c_int, [vp, C.c_int, dp, C.POINTER(C.c_int64), dp]),
        "cnpint_kernel_name": (C.c_char_p, [C.c_int]),
        "cnpint_set_time_dependence": (C.c_int, [vp, dp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _ptr(t) -> int:
    return int(t.data_ptr())


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


@dataclass
class OperatorSpec:
    """Spatial operator L_h (not multiplied by τ), mirrors cnpint_operator."""
    dim: int
    nx: int
    ny: int = 1
    toeplitz: bool = True
    sub: Optional[np.ndarray] = None
    diag: Optional[np.ndarray] = None
    sup: Optional[np.ndarray] = None
    xs: float = 0.0
    xd: float = 0.0
    xu: float = 0.0
    ys: float = 0.0
    yd: float = 0.0
    yu: float = 0.0
    shift: float = 0.0

    def to_c(self):
        keep = []
        op = Operator(self.dim, self.nx, self.ny if self.dim == 2 else 1, int(self.toeplitz), None, None, None,
                      self.xs, self.xd, self.xu, self.ys, self.yd, self.yu, self.shift)
        if self.dim == 1 and not self.toeplitz:
            for name in ("sub", "diag", "sup"):
                arr = np.ascontiguousarray(getattr(self, name), dtype=np.float64)
                keep.append(arr)
                setattr(op, name, arr.ctypes.data_as(C.POINTER(C.c_double)))
        return op, keep


class Solver:
    """One cnpint handle: N time steps on [0, T], α, operator, GMRES basis for restart_max."""

    def __init__(self, N: int, T: float, alpha: float, op: OperatorSpec, restart_max: int = 0, device=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("cnpint needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        self.N, self.T, self.alpha, self.op, self.restart_max = N, T, alpha, op, restart_max
        self.device = torch.device("cuda") if device is None else torch.device(device)
        cop, self._keep = op.to_c()
        nbytes = self.lib.cnpint_workspace_bytes(N, C.byref(cop), restart_max)
        if nbytes == 0:
            raise CnpintError(EINVAL, "cnpint_workspace_bytes rejected the arguments")
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        base = _ptr(self.workspace)
        aligned = (base + 255) // 256 * 256
        h = C.c_void_p()
        st = self.lib.cnpint_create(C.byref(h), N, T, alpha, C.byref(cop), restart_max, C.c_void_p(aligned),
                                    nbytes, _stream())
        if st != OK:
            raise CnpintError(st, "cnpint_create failed")
        self.h = h
        self.ld = int(self.lib.cnpint_ld(h))
        self.vec_elems = int(self.lib.cnpint_vec_elems(h))
        self.spec_elems = int(self.lib.cnpint_spec_elems(h))
        self.ny = op.ny if op.dim == 2 else 1
        self.nx = op.nx

    # ---------------------------------------------------------------- helpers
    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            self.lib.cnpint_destroy(h)
            self.h = None

    def _check(self, st: int, what: str):
        if st != OK:
            msg = self.lib.cnpint_last_error(self.h)
            raise CnpintError(st, f"{what}: {msg.decode() if msg else ''}")

    def _sync_stream(self):
        self.lib.cnpint_set_stream(self.h, _stream())

    @property
    def padded_shape(self):
        return (self.N, self.ld) if self.op.dim == 1 else (self.N, self.ny, self.ld)

    def empty(self):
        import torch
        return torch.zeros(self.padded_shape, dtype=torch.float64, device=self.device)

    def empty_spec(self):
        import torch
        return torch.zeros((self.N // 2 + 1, self.ny * self.ld, 2), dtype=torch.float64, device=self.device)

    def to_device(self, a: np.ndarray):
        """numpy (N, m) / (N, n, n) → zero-padded device tensor."""
        import torch
        t = self.empty()
        t[..., : self.nx] = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self.device)
        return t

    def to_host(self, t) -> np.ndarray:
        return t[..., : self.nx].detach().cpu().numpy().copy()

    # ---------------------------------------------------------------- ABI calls
    def apply_A(self, u, y):
        self._sync_stream()
        self._check(self.lib.cnpint_apply_A(self.h, C.c_void_p(_ptr(u)), C.c_void_p(_ptr(y))), "apply_A")

    def apply_P(self, z, v):
        self._sync_stream()
        self._check(self.lib.cnpint_apply_P(self.h, C.c_void_p(_ptr(z)), C.c_void_p(_ptr(v))), "apply_P")

    def apply_Pinv(self, v, z):
        self._sync_stream()
        self._check(self.lib.cnpint_apply_Pinv(self.h, C.c_void_p(_ptr(v)), C.c_void_p(_ptr(z))), "apply_Pinv")

    def time_fft(self, v, what):
        self._sync_stream()
        self._check(self.lib.cnpint_time_fft(self.h, C.c_void_p(_ptr(v)), C.c_void_p(_ptr(what))), "time_fft")

    def shifted_solve(self, what, zhat):
        self._sync_stream()
        self._check(self.lib.cnpint_shifted_solve(self.h, C.c_void_p(_ptr(what)), C.c_void_p(_ptr(zhat))),
                    "shifted_solve")

    def time_ifft(self, zhat, z):
        self._sync_stream()
        self._check(self.lib.cnpint_time_ifft(self.h, C.c_void_p(_ptr(zhat)), C.c_void_p(_ptr(z))), "time_ifft")

    def gmres(self, b, u, tol: float, restart: int, maxit: int = 1000, history_cap: int = 1000,
              side: str = "right"):
        """cnpint_gmres (side="right", the paper's §5 solver) or cnpint_gmres_left (side="left", the
        §4 / Theorem 4.5 setting; the report adds relres_prec = ||P⁻¹(b − 𝓜u)||/||P⁻¹b||)."""
        if side not in ("right", "left"):
            raise ValueError(f"side must be 'right' or 'left', got {side!r}")
        self._sync_stream()
        hist = (C.c_double * history_cap)()
        rep = GmresReport(0, 0, 0, 0.0, 0.0, 0.0, C.cast(hist, C.POINTER(C.c_double)), history_cap, float("nan"))
        fn = self.lib.cnpint_gmres if side == "right" else self.lib.cnpint_gmres_left
        st = fn(self.h, C.c_void_p(_ptr(b)), C.c_void_p(_ptr(u)), tol, restart, maxit, C.byref(rep))
        if st not in (OK, ENOCONV):
            self._check(st, "gmres" if side == "right" else "gmres_left")
        out = {"status": STATUS[st], "iterations": rep.iterations, "restarts": rep.restarts,
               "converged": bool(rep.converged), "relres_est": rep.relres_est, "relres_true": rep.relres_true,
               "seconds": rep.seconds, "history": [hist[i] for i in range(min(rep.iterations, history_cap))]}
        if side == "left":
            out["relres_prec"] = rep.relres_prec
        return out

    # host-buffer (end-to-end) variants: packed numpy arrays
    def apply_Pinv_host(self, v: np.ndarray, z: Optional[np.ndarray] = None) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64)
        z = np.empty_like(v) if z is None else z
        self._sync_stream()
        self._check(self.lib.cnpint_apply_Pinv_host(self.h, v.ctypes.data_as(C.POINTER(C.c_double)),
                                                    z.ctypes.data_as(C.POINTER(C.c_double))), "apply_Pinv_host")
        return z

    def apply_A_host(self, u: np.ndarray, y: Optional[np.ndarray] = None) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float64)
        y = np.empty_like(u) if y is None else y
        self._sync_stream()
        self._check(self.lib.cnpint_apply_A_host(self.h, u.ctypes.data_as(C.POINTER(C.c_double)),
                                                 y.ctypes.data_as(C.POINTER(C.c_double))), "apply_A_host")
        return y

    def gmres_host(self, b: np.ndarray, tol: float, restart: int, maxit: int = 1000, u: Optional[np.ndarray] = None):
        b = np.ascontiguousarray(b, dtype=np.float64)
        u = np.empty_like(b) if u is None else u
        self._sync_stream()
        rep = GmresReport(0, 0, 0, 0.0, 0.0, 0.0, None, 0, float("nan"))
        st = self.lib.cnpint_gmres_host(self.h, b.ctypes.data_as(C.POINTER(C.c_double)),
                                        u.ctypes.data_as(C.POINTER(C.c_double)), tol, restart, maxit, C.byref(rep))
        if st not in (OK, ENOCONV):
            self._check(st, "gmres_host")
        return u, {"status": STATUS[st], "iterations": rep.iterations, "converged": bool(rep.converged),
                   "relres_true": rep.relres_true, "seconds": rep.seconds}

    def device_status(self) -> int:
        self._sync_stream()
        return int(self.lib.cnpint_device_status(self.h))

    def launch_count(self) -> int:
        return int(self.lib.cnpint_launch_count(self.h))

    def profile_enable(self, on: bool = True):
        self._sync_stream()
        self._check(self.lib.cnpint_profile_enable(self.h, int(on)), "profile_enable")

    def profile_read(self):
        """{kernel class: (ms_total, launches, algorithmic_bytes)} for classes with launches."""
        out = {}
        kid = 0
        while True:
            name = self.lib.cnpint_kernel_name(kid)
            if not name:
                break
            ms, n, by = C.c_double(), C.c_int64(), C.c_double()
            self._check(self.lib.cnpint_profile_read(self.h, kid, C.byref(ms), C.byref(n), C.byref(by)),
                        "profile_read")
            if n.value:
                out[name.decode()] = (ms.value, n.value, by.value)
            kid += 1
        return out

    def set_time_dependence(self, d_half: Optional[np.ndarray]):
        """𝓛(t) = d(t)𝓛 with the N values d(t_{t+½}) (None: constant operator)."""
        self._sync_stream()
        if d_half is None:
            self._check(self.lib.cnpint_set_time_dependence(self.h, None), "set_time_dependence")
            return
        d = np.ascontiguousarray(d_half, dtype=np.float64)
        if d.shape != (self.N,):
            raise CnpintError(EINVAL, f"d_half must have shape ({self.N},)")
        self._check(self.lib.cnpint_set_time_dependence(self.h, d.ctypes.data_as(C.POINTER(C.c_double))),
                    "set_time_dependence")

    def set_debug(self, flags: int):
        self._sync_stream()
        self._check(self.lib.cnpint_set_debug(self.h, flags), "set_debug")


def stream_copy(src, dst):
    lib = load_library()
    st = lib.cnpint_stream_copy(C.c_void_p(_ptr(src)), C.c_void_p(_ptr(dst)), src.numel(), _stream())
    if st != OK:
        raise CnpintError(st, "stream_copy")
