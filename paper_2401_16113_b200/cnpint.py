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
           "cnpint_profile_read", "cnpint_kernel_name", "cnpint_set_time_dependence", "cnpint_gmres_left",
           "cnpint_krylov_basis", "cnpint_peak_kernel",
           "cnpint_shard_workspace_bytes", "cnpint_shard_create", "cnpint_shard_set_collective", "cnpint_shard_buffers",
           "cnpint_shard_apply_Pinv", "cnpint_shard_apply_A", "cnpint_shard_gmres", "cnpint_shard_pinv_begin",
           "cnpint_shard_pinv_end", "cnpint_shard_halo_begin", "cnpint_shard_apply_A_end",
           "cnpint_shard_spike_ends_host", "cnpint_shard_reduced_host", "cnpint_gmres_host_batch"]


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

# int (*)(void* user, int op, const double* d_send, double* d_recv, size_t count, void* cuda_stream)
COLLECTIVE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


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
        "cnpint_krylov_basis": (C.c_int, [vp, C.c_int, C.POINTER(C.c_void_p), dp, C.POINTER(C.c_int)]),
        "cnpint_peak_kernel": (C.c_int, [C.c_int, vp, C.c_int, vp, dp]),
        "cnpint_shard_workspace_bytes": (C.c_size_t, [C.c_int, C.POINTER(Operator), C.c_int, C.POINTER(C.c_int), C.c_int,
                                                      C.c_int]),
        "cnpint_shard_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_double, C.c_double, C.POINTER(Operator),
                                          C.c_int, C.POINTER(C.c_int), C.c_int, C.c_int, vp, C.c_size_t, vp]),
        "cnpint_shard_set_collective": (C.c_int, [vp, COLLECTIVE_FN, vp]),
        "cnpint_shard_buffers": (C.c_int, [vp] + [C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)] * 2),
        "cnpint_shard_apply_Pinv": (C.c_int, [vp, vp, vp]), "cnpint_shard_apply_A": (C.c_int, [vp, vp, vp]),
        "cnpint_shard_gmres": (C.c_int, [vp, vp, vp, C.c_double, C.c_int, C.c_int, C.POINTER(GmresReport)]),
        "cnpint_shard_pinv_begin": (C.c_int, [vp, vp]), "cnpint_shard_pinv_end": (C.c_int, [vp, vp]),
        "cnpint_shard_halo_begin": (C.c_int, [vp, vp]), "cnpint_shard_apply_A_end": (C.c_int, [vp, vp, vp]),
        "cnpint_shard_spike_ends_host": (C.c_int, [C.c_int, C.c_double, C.c_double, C.POINTER(Operator), C.c_int,
                                                   C.POINTER(C.c_int), dp, dp]),
        "cnpint_shard_reduced_host": (C.c_int, [C.c_int, C.c_int, C.c_int, dp, dp, dp, dp]),
        "cnpint_gmres_host_batch": (C.c_int, [vp, C.c_int, C.POINTER(dp), C.POINTER(dp), C.c_double, C.c_int, C.c_int,
                                              vp, C.POINTER(GmresReport)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _ptr(t) -> int:
    return int(t.data_ptr())


def _stream(device=None):
    import torch
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


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
        dev = torch.device("cuda") if device is None else torch.device(device)
        if dev.type != "cuda":
            raise ValueError(f"cnpint needs a CUDA device, got {dev}")
        # a concrete index: the handle lives on one device (its stream, workspace and kernel attributes)
        self.device = torch.device("cuda", torch.cuda.current_device() if dev.index is None else dev.index)
        cop, self._keep = op.to_c()
        nbytes = self.lib.cnpint_workspace_bytes(N, C.byref(cop), restart_max)
        if nbytes == 0:
            raise CnpintError(EINVAL, "cnpint_workspace_bytes rejected the arguments")
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        base = _ptr(self.workspace)
        aligned = (base + 255) // 256 * 256
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            st = self.lib.cnpint_create(C.byref(h), N, T, alpha, C.byref(cop), restart_max, C.c_void_p(aligned),
                                        nbytes, _stream(self.device))
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
        self.lib.cnpint_set_stream(self.h, _stream(self.device))

    def _on_device(self):
        """Every ABI call runs with the handle's device current (kernels launch on its stream)."""
        import torch
        return torch.cuda.device(self.device)

    def _dev(self, t, name: str, elems: int):
        """Device pointer of t after checking what the C side cannot: a contiguous float64 CUDA
        tensor on the handle's device holding at least `elems` doubles (the padded layout)."""
        import torch
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{name} must be a torch.Tensor, got {type(t).__name__}")
        if t.dtype != torch.float64:
            raise CnpintError(EINVAL, f"{name} must be float64, got {t.dtype}")
        if t.device != self.device:
            raise CnpintError(EINVAL, f"{name} is on {t.device}, the handle on {self.device}")
        if not t.is_contiguous():
            raise CnpintError(EINVAL, f"{name} must be contiguous")
        if t.numel() < elems:
            raise CnpintError(EINVAL, f"{name} holds {t.numel()} doubles < {elems} (padded shape "
                                      f"{self.padded_shape})")
        return C.c_void_p(_ptr(t))

    def _vec(self, t, name: str):
        return self._dev(t, name, self.vec_elems)

    def _spec(self, t, name: str):
        return self._dev(t, name, 2 * self.spec_elems)

    def _host_in(self, a, name: str) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.float64)
        if a.shape != self.host_shape:
            raise CnpintError(EINVAL, f"{name} has shape {a.shape}, expected {self.host_shape}")
        return a

    def _host_out(self, a, name: str) -> np.ndarray:
        if a is None:
            return np.empty(self.host_shape, dtype=np.float64)
        if not isinstance(a, np.ndarray) or a.dtype != np.float64 or a.shape != self.host_shape \
                or not a.flags.c_contiguous or not a.flags.writeable:
            raise CnpintError(EINVAL, f"{name} must be a writeable C-contiguous float64 array of shape "
                                      f"{self.host_shape}")
        return a

    @property
    def host_shape(self):
        """Packed host layout of the *_host calls: (N, nx) in 1D, (N, ny, nx) in 2D."""
        return (self.N, self.nx) if self.op.dim == 1 else (self.N, self.ny, self.nx)

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
        pa, pb = self._vec(u, "u"), self._vec(y, "y")
        with self._on_device():
            self._sync_stream()
            self._check(self.lib.cnpint_apply_A(self.h, pa, pb), "apply_A")

    def apply_P(self, z, v):
        pa, pb = self._vec(z, "z"), self._vec(v, "v")
        with self._on_device():
            self._sync_stream()
            self._check(self.lib.cnpint_apply_P(self.h, pa, pb), "apply_P")

    def apply_Pinv(self, v, z):
        pa, pb = self._vec(v, "v"), self._vec(z, "z")
        with self._on_device():
            self._sync_stream()
            self._check(self.lib.cnpint_apply_Pinv(self.h, pa, pb), "apply_Pinv")

    def time_fft(self, v, what):
        pa, pb = self._vec(v, "v"), self._spec(what, "what")
        with self._on_device():
            self._sync_stream()
            self._check(self.lib.cnpint_time_fft(self.h, pa, pb), "time_fft")

    def shifted_solve(self, what, zhat):
        pa, pb = self._spec(what, "what"), self._spec(zhat, "zhat")
        with self._on_device():
            self._sync_stream()
            self._check(self.lib.cnpint_shifted_solve(self.h, pa, pb), "shifted_solve")

    def time_ifft(self, zhat, z):
        pa, pb = self._spec(zhat, "zhat"), self._vec(z, "z")
        with self._on_device():
            self._sync_stream()
            self._check(self.lib.cnpint_time_ifft(self.h, pa, pb), "time_ifft")

    def gmres(self, b, u, tol: float, restart: int, maxit: int = 1000, history_cap: int = 1000,
              side: str = "right"):
        """cnpint_gmres (side="right", the paper's §5 solver) or cnpint_gmres_left (side="left", the
        §4 / Theorem 4.5 setting; the report adds relres_prec = ||P⁻¹(b − 𝓜u)||/||P⁻¹b||)."""
        if side not in ("right", "left"):
            raise ValueError(f"side must be 'right' or 'left', got {side!r}")
        pb, pu = self._vec(b, "b"), self._vec(u, "u")
        hist = (C.c_double * history_cap)()
        rep = GmresReport(0, 0, 0, 0.0, 0.0, 0.0, C.cast(hist, C.POINTER(C.c_double)), history_cap, float("nan"))
        fn = self.lib.cnpint_gmres if side == "right" else self.lib.cnpint_gmres_left
        with self._on_device():
            self._sync_stream()
            st = fn(self.h, pb, pu, tol, restart, maxit, C.byref(rep))
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
        v = self._host_in(v, "v")
        z = self._host_out(z, "z")
        with self._on_device():
            self._sync_stream()
            self._check(self.lib.cnpint_apply_Pinv_host(self.h, v.ctypes.data_as(C.POINTER(C.c_double)),
                                                        z.ctypes.data_as(C.POINTER(C.c_double))), "apply_Pinv_host")
        return z

    def apply_A_host(self, u: np.ndarray, y: Optional[np.ndarray] = None) -> np.ndarray:
        u = self._host_in(u, "u")
        y = self._host_out(y, "y")
        with self._on_device():
            self._sync_stream()
            self._check(self.lib.cnpint_apply_A_host(self.h, u.ctypes.data_as(C.POINTER(C.c_double)),
                                                     y.ctypes.data_as(C.POINTER(C.c_double))), "apply_A_host")
        return y

    def gmres_host(self, b: np.ndarray, tol: float, restart: int, maxit: int = 1000, u: Optional[np.ndarray] = None):
        b = self._host_in(b, "b")
        u = self._host_out(u, "u")
        rep = GmresReport(0, 0, 0, 0.0, 0.0, 0.0, None, 0, float("nan"))
        with self._on_device():
            self._sync_stream()
            st = self.lib.cnpint_gmres_host(self.h, b.ctypes.data_as(C.POINTER(C.c_double)),
                                            u.ctypes.data_as(C.POINTER(C.c_double)), tol, restart, maxit,
                                            C.byref(rep))
        if st not in (OK, ENOCONV):
            self._check(st, "gmres_host")
        return u, {"status": STATUS[st], "iterations": rep.iterations, "converged": bool(rep.converged),
                   "relres_true": rep.relres_true, "seconds": rep.seconds}

    def gmres_host_batch(self, bs, us, tol: float, restart: int, maxit: int = 1000, stage=None):
        """cnpint_gmres_host_batch over the host arrays bs → us (lists of packed float64 arrays, pinned for
        overlap); stage: optional device scratch of 4·vec_elems doubles (allocated if None)."""
        import torch
        bs = [self._host_in(b, "b") for b in bs]
        us = [self._host_out(u, "u") for u in us]
        if len(bs) != len(us) or not bs:
            raise CnpintError(EINVAL, "need as many outputs as right-hand sides")
        if stage is None:
            stage = torch.empty(4 * self.vec_elems, dtype=torch.float64, device=self.device)
        ps = self._dev(stage, "stage", 4 * self.vec_elems)
        dp = C.POINTER(C.c_double)
        hb = (dp * len(bs))(*[b.ctypes.data_as(dp) for b in bs])
        hu = (dp * len(us))(*[u.ctypes.data_as(dp) for u in us])
        reps = (GmresReport * len(bs))()
        with self._on_device():
            self._sync_stream()
            st = self.lib.cnpint_gmres_host_batch(self.h, len(bs), hb, hu, tol, restart, maxit, ps, reps)
        if st not in (OK, ENOCONV):
            self._check(st, "gmres_host_batch")
        return [{"iterations": r.iterations, "converged": bool(r.converged), "relres_true": r.relres_true}
                for r in reps]

    def device_status(self) -> int:
        with self._on_device():
            self._sync_stream()
            return int(self.lib.cnpint_device_status(self.h))

    def launch_count(self) -> int:
        return int(self.lib.cnpint_launch_count(self.h))

    def profile_enable(self, on: bool = True):
        with self._on_device():
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
        d = None
        if d_half is not None:
            d = np.ascontiguousarray(d_half, dtype=np.float64)
            if d.shape != (self.N,):
                raise CnpintError(EINVAL, f"d_half must have shape ({self.N},)")
        with self._on_device():
            self._sync_stream()
            self._check(self.lib.cnpint_set_time_dependence(
                self.h, None if d is None else d.ctypes.data_as(C.POINTER(C.c_double))), "set_time_dependence")

    def krylov_basis(self):
        """The last GMRES cycle's basis as (list of torch views Ṽ_i, list of scales s_i), v_i = s_iṼ_i
        (test hook for orthogonality measurements; the views alias the workspace / the caller's b)."""
        import torch
        cnt = C.c_int(0)
        with self._on_device():
            self._sync_stream()
            self.lib.cnpint_krylov_basis(self.h, 0, None, None, C.byref(cnt))
            vecs, scales = [], []
            for i in range(cnt.value):
                p, s = C.c_void_p(), C.c_double()
                self._check(self.lib.cnpint_krylov_basis(self.h, i, C.byref(p), C.byref(s), None), "krylov_basis")
                base = _ptr(self.workspace)
                if p.value >= base and p.value < base + self.workspace.numel():
                    off = (p.value - base) // 8
                    ws = self.workspace.view(torch.float64) if (base % 8 == 0) else None
                    vecs.append(ws[off:off + self.vec_elems].view(self.padded_shape))
                else:
                    vecs.append(None)   # the caller's b (first cycle): the caller holds it
                scales.append(s.value)
        return vecs, scales

    def set_debug(self, flags: int):
        with self._on_device():
            self._sync_stream()
            self._check(self.lib.cnpint_set_debug(self.h, flags), "set_debug")


def peak_kernel(kind: int, out, iters: int) -> float:
    """Enqueue the fp64 FMA (kind 0) / DMMA (kind 1) ceiling kernel on torch's current stream; returns
    the flops of the launch (the caller times it with CUDA events)."""
    lib = load_library()
    fl = C.c_double()
    st = lib.cnpint_peak_kernel(kind, C.c_void_p(_ptr(out)), iters, _stream(), C.byref(fl))
    if st != OK:
        raise CnpintError(st, "peak_kernel")
    return fl.value


def stream_copy(src, dst):
    lib = load_library()
    st = lib.cnpint_stream_copy(C.c_void_p(_ptr(src)), C.c_void_p(_ptr(dst)), src.numel(), _stream())
    if st != OK:
        raise CnpintError(st, "stream_copy")
