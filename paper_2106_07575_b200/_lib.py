"""ctypes binding of libptyger (include/ptyger.h): argument marshalling only.

Every step of the CG iteration runs in the library's CUDA kernels; there is no Python or CPU
fallback.  If libptyger.so is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PTYGER_LIB: an alternative build of the same library (A/B experiments); default: the in-tree build
LIB_PATH = os.environ.get("PTYGER_LIB") or os.path.join(_HERE, "libptyger.so")

PTYGER_OK = 0
STATUS = {0: "OK", 2: "E_ARG", 3: "E_DATA", 4: "E_NUMERIC", 5: "E_CUDA", 6: "E_NCCL", 7: "E_OOM", 8: "E_STATE"}
DIR_DY, DIR_DY_REAL, DIR_FR, DIR_PR, DIR_GD = 0, 1, 2, 3, 4
EST_ML, EST_LS = 0, 1
TRANSPORT_NCCL, TRANSPORT_P2P = 0, 1


class PtygerError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [("gamma0", C.c_double), ("tau", C.c_double), ("t", C.c_double), ("eps", C.c_double),
                ("max_shrinks", C.c_int32), ("direction", C.c_int32), ("ls_batch", C.c_int32),
                ("estimator", C.c_int32),
                ("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32), ("nccl_id", C.c_void_p),
                ("transport", C.c_int32)]


class Trace(C.Structure):
    _fields_ = [("iter", C.c_int32), ("shrinks", C.c_int32), ("restarted", C.c_int32), ("stalled", C.c_int32),
                ("F", C.c_double), ("gamma", C.c_double), ("alpha_re", C.c_double), ("alpha_im", C.c_double),
                ("grad_norm", C.c_double), ("step_norm", C.c_double),
                ("ms_grad", C.c_float), ("ms_dir", C.c_float), ("ms_ls", C.c_float), ("ms_update", C.c_float),
                ("ms_comm", C.c_float), ("ls_passes", C.c_int32), ("ls_exact_passes", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(LIB_PATH)
    P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "ptyger_config_default": (None, [C.POINTER(Config)]),
        "ptyger_init": (I32, [C.POINTER(P), C.POINTER(Config), P, I64, I64, P, I32, P, I64, P]),
        "ptyger_init_subpixel": (I32, [C.POINTER(P), C.POINTER(Config), P, I64, I64, P, I32, P, I64, P]),
        "ptyger_partition_subpixel": (I32, [P, I64, I64, I32, I32, P, P]),
        "ptyger_ipc_handle": (I32, [P, P]),
        "ptyger_ipc_connect": (I32, [P, P]),
        "ptyger_cg_iterate": (I32, [P, I32, P]),
        "ptyger_cg_launch": (I32, [P, I32]),
        "ptyger_cg_wait": (I32, [P, P]),
        "ptyger_stream": (P, [P]),
        "ptyger_get_object": (I32, [P, P]),
        "ptyger_get_gradient": (I32, [P, P]),
        "ptyger_get_farfield": (I32, [P, P]),
        "ptyger_get_state": (I32, [P, P, P, P, P, P]),
        "ptyger_set_state": (I32, [P, P, P, P, I32]),
        "ptyger_get_ls_partials": (I32, [P, P, P, I32, P]),
        "ptyger_partition": (I32, [P, I64, I64, I32, I32, P, P]),
        "ptyger_round_positions": (I32, [P, I64, P]),
        "ptyger_fft2": (I32, [P, P, I32, I64, I32, P]),
        "ptyger_nccl_unique_id": (I32, [P]),
        "ptyger_last_error": (C.c_char_p, [P]),
        "ptyger_kernel_launches": (I64, [P]),
        "ptyger_last_iterate_ms": (C.c_float, [P]),
        "ptyger_kernel_times": (I32, [P, P, P, I32]),
        "ptyger_fp32_peak": (I32, [I32, I32, P]),
        "ptyger_destroy": (None, [P]),
        "ptyger_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def last_error(ctx=None) -> str:
    s = lib.ptyger_last_error(ctx)
    return s.decode() if s else ""


def _check(status: int, ctx=None):
    if status != PTYGER_OK:
        raise PtygerError(status, last_error(ctx))


def default_config(**kw) -> Config:
    c = Config()
    lib.ptyger_config_default(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def _ptr(a):
    """Host numpy array or torch tensor (host or CUDA) -> (pointer, keepalive)."""
    if a is None:
        return None, None
    if hasattr(a, "data_ptr"):           # torch tensor
        if not a.is_contiguous():
            a = a.contiguous()
        return a.data_ptr(), a
    a = np.ascontiguousarray(a)
    return a.ctypes.data, a


def as_c64(a):
    """complex array -> interleaved float32 view/buffer; torch tensors pass through."""
    if hasattr(a, "data_ptr"):
        import torch
        if a.is_complex():
            return torch.view_as_real(a.to(torch.complex64).contiguous())
        return a.float().contiguous()
    a = np.asarray(a)
    if np.iscomplexobj(a):
        return np.ascontiguousarray(a.astype(np.complex64)).view(np.float32)
    return np.ascontiguousarray(a, dtype=np.float32)


def partition(scan, H: int, N: int, P: int):
    scan = np.ascontiguousarray(scan, dtype=np.int32)
    n = len(scan)
    rank = np.zeros(n, np.int32)
    rows = np.zeros((P, 6), np.int64)
    _check(lib.ptyger_partition(scan.ctypes.data, n, H, N, P, rank.ctypes.data, rows.ctypes.data))
    return rank, rows


def partition_subpixel(scan, H: int, N: int, P: int):
    scan = np.ascontiguousarray(scan, dtype=np.float32)
    n = len(scan)
    rank = np.zeros(n, np.int32)
    rows = np.zeros((P, 6), np.int64)
    _check(lib.ptyger_partition_subpixel(scan.ctypes.data, n, H, N, P, rank.ctypes.data, rows.ctypes.data))
    return rank, rows


def round_positions(raw):
    raw = np.ascontiguousarray(raw, dtype=np.float32)
    out = np.zeros(raw.shape, np.int32)
    _check(lib.ptyger_round_positions(raw.ctypes.data, len(raw), out.ctypes.data))
    return out


def fft2(x, inverse: bool = False, out=None):
    """Library batched unitary 2-D FFT on a CUDA complex64 tensor (..., N, N)."""
    import torch
    assert x.is_cuda and x.dtype == torch.complex64
    x = x.contiguous()
    N = x.shape[-1]
    batch = x.numel() // (N * N)
    if out is None:
        out = torch.empty_like(x)
    stream = torch.cuda.current_stream(x.device).cuda_stream
    _check(lib.ptyger_fft2(x.data_ptr(), out.data_ptr(), N, batch, int(inverse), stream))
    return out


def fp32_peak(device: int = 0, paired: bool = True) -> float:
    """Measured FP32 FMA-pipe peak of the device in TFLOP/s (ptyger_fp32_peak)."""
    out = C.c_double()
    _check(lib.ptyger_fp32_peak(device, int(paired), C.byref(out)))
    return float(out.value)


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib.ptyger_nccl_unique_id(buf))
    return bytes(buf)


class Ptyger:
    """One reconstruction problem resident on one GPU (or one stripe of it when world > 1).

    Wraps ptyger_init / ptyger_cg_iterate / ptyger_get_object (Alg.1)."""

    def __init__(self, obj, probe, scan, d, config: Config | None = None, **cfg):
        self.cfg = config if config is not None else default_config(**cfg)
        o = as_c64(obj)
        p = as_c64(probe)
        self.H, self.W = (o.shape[0], o.shape[1]) if o.ndim == 3 else (obj.shape[0], obj.shape[1])
        self.N = int(probe.shape[0])
        # a floating-point scan array selects the fractional-position (bilinear window) entry point
        if hasattr(scan, "data_ptr"):   # torch tensor (host or CUDA): positions are read on the host
            scan = scan.detach().cpu().numpy()
        self.subpixel = np.issubdtype(np.asarray(scan).dtype, np.floating)
        sc = np.ascontiguousarray(np.asarray(scan), dtype=np.float32 if self.subpixel else np.int32)
        self.n = len(sc)
        if hasattr(d, "data_ptr"):      # torch tensor: float32, contiguous, on its own device
            dd = d.detach().to(dtype=__import__("torch").float32).contiguous()
            nel = dd.numel()
        else:
            dd = np.ascontiguousarray(d, dtype=np.float32)
            nel = dd.size
        if nel != self.n * self.N * self.N:
            raise PtygerError(3, f"intensities hold {nel} values, expected n*N*N = {self.n * self.N * self.N}")
        po, ko = _ptr(o)
        pp, kp = _ptr(p)
        pd, kd = _ptr(dd)
        self.ctx = C.c_void_p()
        init = lib.ptyger_init_subpixel if self.subpixel else lib.ptyger_init
        st = init(C.byref(self.ctx), C.byref(self.cfg), po, self.H, self.W, pp, self.N, sc.ctypes.data, self.n, pd)
        _check(st, None)
        self.K = self.cfg.ls_batch

    def ipc_handle(self) -> bytes:
        """P2P transport: this rank's 64-byte exchange-window handle (exchange it out of band)."""
        buf = (C.c_char * 64)()
        _check(lib.ptyger_ipc_handle(self.ctx, buf), self.ctx)
        return bytes(buf)

    def ipc_connect(self, handles):
        """P2P transport: all ranks' handles in rank order (list of 64-byte strings)."""
        blob = b"".join(handles)
        assert len(blob) == 64 * self.cfg.world
        buf = (C.c_char * len(blob)).from_buffer_copy(blob)
        _check(lib.ptyger_ipc_connect(self.ctx, buf), self.ctx)

    def close(self):
        if getattr(self, "ctx", None) and self.ctx.value:
            lib.ptyger_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def iterate(self, n_iter: int, traces: bool = True):
        tr = (Trace * max(n_iter, 1))()
        _check(lib.ptyger_cg_iterate(self.ctx, n_iter, tr if traces else None), self.ctx)
        return [tr[i].as_dict() for i in range(n_iter)] if traces else None

    def launch(self, n_iter: int):
        """Enqueue n_iter iterations on the context's stream without waiting (see wait())."""
        self._pending = n_iter
        _check(lib.ptyger_cg_launch(self.ctx, n_iter), self.ctx)

    def wait(self, traces: bool = True):
        n = getattr(self, "_pending", 0)
        self._pending = 0
        tr = (Trace * max(n, 1))()
        _check(lib.ptyger_cg_wait(self.ctx, tr if traces else None), self.ctx)
        return [tr[i].as_dict() for i in range(n)] if traces else None

    def stream(self) -> int:
        """cudaStream_t of the context (e.g. for torch.cuda.ExternalStream)."""
        return int(lib.ptyger_stream(self.ctx) or 0)

    def _obj_buf(self):
        return np.empty((self.H, self.W), np.complex64)

    def get_object(self, out=None):
        """psi_m as (H, W) complex64; `out` may be a caller buffer (e.g. a pinned-memory view, which
        makes the device-to-host copy run at full link speed)."""
        if out is None:
            out = self._obj_buf()
        assert out.dtype == np.complex64 and out.shape == (self.H, self.W) and out.flags["C_CONTIGUOUS"]
        _check(lib.ptyger_get_object(self.ctx, out.ctypes.data), self.ctx)
        return out

    def get_gradient(self):
        out = self._obj_buf()
        _check(lib.ptyger_get_gradient(self.ctx, out.ctypes.data), self.ctx)
        return out

    def get_farfield(self, n_local: int | None = None):
        out = np.empty((n_local if n_local is not None else self.n, self.N, self.N), np.complex64)
        _check(lib.ptyger_get_farfield(self.ctx, out.ctypes.data), self.ctx)
        return out

    def get_state(self):
        psi, g, e = self._obj_buf(), self._obj_buf(), self._obj_buf()
        F = C.c_double()
        m = C.c_int32()
        _check(lib.ptyger_get_state(self.ctx, psi.ctypes.data, g.ctypes.data, e.ctypes.data, C.byref(F),
                                    C.byref(m)), self.ctx)
        return psi, g, e, F.value, m.value

    def set_state(self, psi, g_prev=None, eta_prev=None, m: int = 0):
        a = np.ascontiguousarray(psi, dtype=np.complex64)
        b = None if g_prev is None else np.ascontiguousarray(g_prev, dtype=np.complex64)
        c = None if eta_prev is None else np.ascontiguousarray(eta_prev, dtype=np.complex64)
        _check(lib.ptyger_set_state(self.ctx, a.ctypes.data, None if b is None else b.ctypes.data,
                                    None if c is None else c.ctypes.data, m), self.ctx)

    def get_ls_partials(self, K: int = 64, with_bound: bool = False):
        out = np.empty(K, np.float64)
        bnd = np.empty(K, np.float64)
        ne = C.c_int32()
        _check(lib.ptyger_get_ls_partials(self.ctx, out.ctypes.data, bnd.ctypes.data, K, C.byref(ne)), self.ctx)
        return (out[:ne.value], bnd[:ne.value]) if with_bound else out[:ne.value]

    def last_iterate_ms(self) -> float:
        return float(lib.ptyger_last_iterate_ms(self.ctx))

    def kernel_times(self, reset: bool = True):
        """{"k_grad": (total ms, launches), "k_ls": (total ms, launches)} since the last reset."""
        ms = np.zeros(2, np.float64)
        cnt = np.zeros(2, np.int32)
        _check(lib.ptyger_kernel_times(self.ctx, ms.ctypes.data, cnt.ctypes.data, int(reset)), self.ctx)
        return {"k_grad": (float(ms[0]), int(cnt[0])), "k_ls": (float(ms[1]), int(cnt[1]))}

    def kernel_launches(self) -> int:
        return int(lib.ptyger_kernel_launches(self.ctx))


class ViewBatch:
    """3-D ptycho-tomography batch: the rotation views
    are independent 2-D problems, so each view gets its own context (own psi, far fields, alpha,
    gamma) and the batch iterates them back to back on this GPU.  Across GPUs the views are
    sharded with no communication (bench.py --config view3d)."""

    def __init__(self, views, **cfg):
        # views: iterable of (psi0, probe, scan, d)
        self.views = [Ptyger(o, p, s, d, **cfg) for (o, p, s, d) in views]

    def iterate(self, n_iter: int, traces: bool = True):
        """All views' iterations are enqueued before any is waited for: the views' streams overlap."""
        for v in self.views:
            v.launch(n_iter)
        return [v.wait(traces) for v in self.views]

    def last_iterate_ms(self) -> float:
        return sum(v.last_iterate_ms() for v in self.views)

    def kernel_times(self, reset: bool = True):
        """Summed over the views: {"k_grad": (total ms, launches), "k_ls": (total ms, launches)}."""
        out = {"k_grad": (0.0, 0), "k_ls": (0.0, 0)}
        for v in self.views:
            for k, (ms, n) in v.kernel_times(reset).items():
                out[k] = (out[k][0] + ms, out[k][1] + n)
        return out

    def kernel_launches(self) -> int:
        return sum(v.kernel_launches() for v in self.views)

    def close(self):
        for v in self.views:
            v.close()
