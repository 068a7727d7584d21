"""x-sharded 1D handles over torch.distributed (include/cnpint.h "1D
x-sharded handles").

Argument marshalling around the cnpint_shard_* C ABI: the partition of the spatial index into R
contiguous chunks, the collective callback (all-gather of the P_α⁻¹ end values and of the 𝓜u boundary
columns, all-reduce of the GMRES dot products) implemented with torch.distributed (NCCL between GPUs;
gloo for the host-side tests), and views of the exchange buffers inside the caller-owned workspace.
Every arithmetic step runs in libcnpint.so's kernels.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from .cnpint import (COLLECTIVE_FN, EINVAL, ENOCONV, OK, STATUS, CnpintError, GmresReport, OperatorSpec,
                     load_library, _ptr, _stream)


def partition(m: int, R: int) -> list:
    """Chunk bounds x0[0..R] of m rows over R ranks, as equal as possible (the first m mod R chunks one
    row longer); every chunk needs >= 2 rows."""
    if R < 1 or m < 2 * R:
        raise ValueError(f"cannot split {m} rows into {R} chunks of >= 2")
    q, rem = divmod(m, R)
    x0 = [0]
    for r in range(R):
        x0.append(x0[-1] + q + (1 if r < rem else 0))
    return x0


class TorchDistComm:
    """The collectives of a sharded handle over a torch.distributed process group (NCCL for CUDA
    tensors, gloo for CPU tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group

    def allgather(self, send, recv):
        self.dist.all_gather_into_tensor(recv, send, group=self.group)

    def allreduce_(self, buf):
        self.dist.all_reduce(buf, op=self.dist.ReduceOp.SUM, group=self.group)


class ShardSolver:
    """Rank `rank` of an R-way x-sharded AaO system (1D operator `op`, global size op.nx)."""

    def __init__(self, N: int, T: float, alpha: float, op: OperatorSpec, rank: int, world: int,
                 restart_max: int = 0, device=None, comm=None, x0: Optional[list] = None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("cnpint needs a CUDA device (no CPU fallback)")
        if op.dim != 1:
            raise ValueError("sharding is for 1D operators")
        self.lib = load_library()
        self.N, self.rank, self.world, self.op = N, rank, world, op
        self.x0 = list(x0) if x0 is not None else partition(op.nx, world)
        self.c0, self.c1 = self.x0[rank], self.x0[rank + 1]
        self.nx = self.c1 - self.c0
        dev = torch.device("cuda") if device is None else torch.device(device)
        self.device = torch.device("cuda", torch.cuda.current_device() if dev.index is None else dev.index)
        self.comm = comm
        cop, self._keep = op.to_c()
        bounds = (C.c_int * (world + 1))(*self.x0)
        nbytes = self.lib.cnpint_shard_workspace_bytes(N, C.byref(cop), world, bounds, rank, restart_max)
        if nbytes == 0:
            raise CnpintError(EINVAL, "cnpint_shard_workspace_bytes rejected the arguments")
        self.workspace = torch.empty((nbytes + 511) // 256 * 256, dtype=torch.uint8, device=self.device)
        base = _ptr(self.workspace)
        self._base = (base + 255) // 256 * 256
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            st = self.lib.cnpint_shard_create(C.byref(h), N, T, alpha, C.byref(cop), world, bounds, rank, restart_max,
                                              C.c_void_p(self._base), nbytes, _stream(self.device))
        if st != OK:
            raise CnpintError(st, "cnpint_shard_create failed")
        self.h = h
        self.ld = int(self.lib.cnpint_ld(h))
        self.vec_elems = int(self.lib.cnpint_vec_elems(h))
        self._ws64 = self.workspace.view(torch.float64)
        self._cb = COLLECTIVE_FN(self._collective)
        self.lib.cnpint_shard_set_collective(h, self._cb, None)
        self.error = None

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            self.lib.cnpint_destroy(h)
            self.h = None

    # ------------------------------------------------------------------ plumbing
    def _view(self, ptr: int, count: int):
        off = ptr - _ptr(self.workspace)
        if off < 0 or off % 8 or off + 8 * count > self.workspace.numel():
            raise CnpintError(EINVAL, "collective buffer outside the workspace")
        return self._ws64[off // 8: off // 8 + count]

    def _collective(self, user, op, send, recv, count, stream):
        try:
            if op == 0:
                self.comm.allgather(self._view(send, count), self._view(recv, count * self.world))
            else:
                self.comm.allreduce_(self._view(send, count))
            return 0
        except Exception as e:  # reported by the C side as a failed collective
            self.error = e
            return 1

    def _check(self, st: int, what: str):
        if st != OK:
            msg = self.lib.cnpint_last_error(self.h)
            raise CnpintError(st, f"{what}: {msg.decode() if msg else ''}"
                                  + (f" ({self.error!r})" if self.error is not None else ""))

    def _on_device(self):
        import torch
        return torch.cuda.device(self.device)

    def _vec(self, t, name):
        import torch
        if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or t.device != self.device \
                or not t.is_contiguous() or t.numel() < self.vec_elems:
            raise CnpintError(EINVAL, f"{name} must be a contiguous float64 tensor on {self.device} of shape "
                                      f"{(self.N, self.ld)}")
        return C.c_void_p(_ptr(t))

    def buffers(self):
        """Views of the exchange buffers: (ends_send, ends_recv, halo_send, halo_recv)."""
        es, er, hs, hr = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        ec, hc = C.c_size_t(), C.c_size_t()
        self._check(self.lib.cnpint_shard_buffers(self.h, C.byref(es), C.byref(er), C.byref(ec), C.byref(hs),
                                                  C.byref(hr), C.byref(hc)), "shard_buffers")
        return (self._view(es.value, ec.value), self._view(er.value, ec.value * self.world),
                self._view(hs.value, hc.value), self._view(hr.value, hc.value * self.world))

    # ------------------------------------------------------------------ vectors (rank-local columns)
    def empty(self):
        import torch
        return torch.zeros((self.N, self.ld), dtype=torch.float64, device=self.device)

    def to_device(self, a_local: np.ndarray):
        import torch
        t = self.empty()
        t[:, : self.nx] = torch.from_numpy(np.ascontiguousarray(a_local, dtype=np.float64)).to(self.device)
        return t

    def to_host(self, t) -> np.ndarray:
        return t[:, : self.nx].detach().cpu().numpy().copy()

    # ------------------------------------------------------------------ ABI calls
    def _call(self, fn, what, *args):
        with self._on_device():
            self.lib.cnpint_set_stream(self.h, _stream(self.device))
            self._check(fn(self.h, *args), what)

    def apply_Pinv(self, v, z):
        self._call(self.lib.cnpint_shard_apply_Pinv, "shard_apply_Pinv", self._vec(v, "v"), self._vec(z, "z"))

    def apply_A(self, u, y):
        self._call(self.lib.cnpint_shard_apply_A, "shard_apply_A", self._vec(u, "u"), self._vec(y, "y"))

    def pinv_begin(self, v):
        self._call(self.lib.cnpint_shard_pinv_begin, "shard_pinv_begin", self._vec(v, "v"))

    def pinv_end(self, z):
        self._call(self.lib.cnpint_shard_pinv_end, "shard_pinv_end", self._vec(z, "z"))

    def halo_begin(self, u):
        self._call(self.lib.cnpint_shard_halo_begin, "shard_halo_begin", self._vec(u, "u"))

    def apply_A_end(self, u, y):
        self._call(self.lib.cnpint_shard_apply_A_end, "shard_apply_A_end", self._vec(u, "u"), self._vec(y, "y"))

    def gmres(self, b, u, tol: float, restart: int, maxit: int = 1000, history_cap: int = 1000):
        hist = (C.c_double * history_cap)()
        rep = GmresReport(0, 0, 0, 0.0, 0.0, 0.0, C.cast(hist, C.POINTER(C.c_double)), history_cap, float("nan"))
        pb, pu = self._vec(b, "b"), self._vec(u, "u")
        with self._on_device():
            self.lib.cnpint_set_stream(self.h, _stream(self.device))
            st = self.lib.cnpint_shard_gmres(self.h, pb, pu, tol, restart, maxit, C.byref(rep))
        if st not in (OK, ENOCONV):
            self._check(st, "shard_gmres")
        return {"status": STATUS[st], "iterations": rep.iterations, "restarts": rep.restarts,
                "converged": bool(rep.converged), "relres_est": rep.relres_est, "relres_true": rep.relres_true,
                "seconds": rep.seconds, "history": [hist[i] for i in range(min(rep.iterations, history_cap))]}

    def device_status(self) -> int:
        with self._on_device():
            self.lib.cnpint_set_stream(self.h, _stream(self.device))
            return int(self.lib.cnpint_device_status(self.h))


# ---------------------------------------------------------------------- host-only partition arithmetic
def spike_ends_host(N: int, T: float, alpha: float, op: OperatorSpec, x0: list):
    """cnpint_shard_spike_ends_host: (red [K][R][4] complex, ab [R][2]) for the chunk bounds x0."""
    lib = load_library()
    R, K = len(x0) - 1, N // 2 + 1
    cop, keep = op.to_c()
    red = np.zeros(K * R * 4 * 2)
    ab = np.zeros(R * 2)
    st = lib.cnpint_shard_spike_ends_host(N, T, alpha, C.byref(cop), R, (C.c_int * (R + 1))(*x0),
                                          red.ctypes.data_as(C.POINTER(C.c_double)),
                                          ab.ctypes.data_as(C.POINTER(C.c_double)))
    if st != OK:
        raise CnpintError(st, "cnpint_shard_spike_ends_host")
    return red.view(np.complex128).reshape(K, R, 4), ab.reshape(R, 2)


def reduced_neighbours_host(red: np.ndarray, ab: np.ndarray, ends_all: np.ndarray, rank: int):
    """cnpint_shard_reduced_host: per frequency (xe_{rank−1}, xs_{rank+1}) from every rank's end values
    ends_all [R][K][2] (complex)."""
    lib = load_library()
    R, K = ends_all.shape[0], ends_all.shape[1]
    red_r = np.ascontiguousarray(red, dtype=np.complex128).view(np.float64)
    ab_r = np.ascontiguousarray(ab, dtype=np.float64)
    ends_r = np.ascontiguousarray(ends_all, dtype=np.complex128).view(np.float64)
    out = np.zeros(K * 4)
    dp = C.POINTER(C.c_double)
    st = lib.cnpint_shard_reduced_host(K, R, rank, red_r.ctypes.data_as(dp), ab_r.ctypes.data_as(dp),
                                       ends_r.ctypes.data_as(dp), out.ctypes.data_as(dp))
    if st != OK:
        raise CnpintError(st, "cnpint_shard_reduced_host")
    return out.view(np.complex128).reshape(K, 2)
