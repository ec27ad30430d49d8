"""ctypes binding of libscurve_b200.so (include/scurve_b200.h).

The product path has no CPU fallback: if the shared library or a CUDA
device is missing, every transform raises.  One context per device is
created lazily and shared; calls are serialised per context by a lock
(a context is not thread-safe, include/scurve_b200.h).
"""

from __future__ import annotations

import contextlib
import contextvars
import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libscurve_b200.so")

SCV_OK = 0
SCV_EINVAL = -1
SCV_ETYPE = -2

_lib = None
_lib_lock = threading.Lock()

_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_LL = ctypes.c_longlong

# name -> argtypes (all return int unless listed in _RESTYPE)
_SIGS = {
    "scv_version": [],
    "scv_create": [_I, ctypes.POINTER(_P)],
    "scv_destroy": [_P],
    "scv_last_error": [_P],
    "scv_workspace_bytes": [_P],
    "scv_trim": [_P],
    "scv_profile": [_P, _I],
    "scv_set_option": [_P, ctypes.c_char_p, _I],
    "scv_launch_count": [_P],
    "scv_profile_report": [_P, ctypes.c_char_p, _I],
    "scv_fp64_peak": [_P, ctypes.POINTER(ctypes.c_double)],
    "scv_dmma_peak": [_P, ctypes.POINTER(ctypes.c_double)],
    "scv_debug_dft": [_P, _I, _I, _I, _P, _P, _P],
    "scv_debug_pfa_maps": [_I, _P, _P],
    "scv_debug_r89_sigma": [_P, _P],
    "scv_debug_pfa_sched": [_I, _P, _P],
    "scv_debug_pipe_stats": [_P, _I],
    "scv_debug_betaq_build": [_P, _I, _I, _P, ctypes.c_longlong, _P],
    "scv_syn_chunk_rows": [_I],
    "scv_betaq_restrict": [_P, _I, _I, _I],
    "scv_halfpi_wedge": [_P, _I, _P, _P],
    "scv_sht_forward": [_P, _I, _I, _I, _P, _P, _P],
    "scv_sht_inverse": [_P, _I, _I, _I, _P, _P, _P],
    "scv_scale_product": [_P, _I, _I, _P, _P, _P, _P, _P],
    "scv_scaling_product": [_P, _I, _I, _P, _P, _P, _P],
    "scv_so3_inverse_curvelet": [_P, _I, _I, _P, _P, _P],
    "scv_so3_forward_curvelet": [_P, _I, _I, _P, _P, _P],
    "scv_so3_inverse_curvelet_slab": [_P, _I, _P, _I, _I, _P, _P],
    "scv_so3_forward_curvelet_slab": [_P, _I, _I, _P, _I, _I, _P, _I, _P],
    "scv_accumulate": [_P, _I, _I, _P, _P, _P, _P, _P],
    "scv_accumulate_scaling": [_P, _I, _I, _P, _P, _P, _P],
    "scv_finish_acc": [_P, _I, _I, _I, _P, _P],
    "scv_map_work_bytes": [_I, _I, _I],
    "scv_analyze": [_P, _I, _I, _I, _I, _P, _P, _P, _P, _I, _P, _P, _P, _P, _LL, _P],
    "scv_synthesize": [_P, _I, _I, _I, _I, _P, _P, _P, _P, _I, _P, _P, _P, _P, _LL, _P],
    "scv_edge_columns": [_P, _I, _D, _P, _P],
    "scv_rotate_to_north": [_P, _I, _D, _P, _P, _P],
    "scv_rotate_from_north": [_P, _I, _D, _P, _P, _P],
    "scv_so3_inverse_general": [_P, _I, _I, _I, _I, _P, _P, _P],
    "scv_so3_forward_general": [_P, _I, _I, _I, _I, _P, _P, _P],
    "scv_abs_max": [_P, _LL, _I, _P, _P, _P, _P],
    "scv_histogram": [_P, _LL, _P, _P, _I, _P, _P, _P],
    "scv_sort_f64": [_P, _LL, _P, _P, ctypes.POINTER(_I), _P],
    "scv_gini_sums": [_P, _LL, _P, _P, _P],
}
_RESTYPE = {"scv_last_error": ctypes.c_char_p, "scv_workspace_bytes": ctypes.c_longlong,
            "scv_launch_count": ctypes.c_longlong, "scv_map_work_bytes": ctypes.c_longlong}

EXPORTED = tuple(_SIGS)


def load_library(path: str | None = None):
    """Load (once) and type the C ABI.  Raises if the library is missing."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        p = path or os.environ.get("SCV_LIB") or LIB_PATH
        if not os.path.exists(p):
            raise RuntimeError(
                f"{p} not found: build the CUDA library first "
                "(python -m paper_1511_05578_b200.build); there is no CPU fallback")
        lib = ctypes.CDLL(p)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, ctypes.c_int)
        _lib = lib
        return lib


class Context:
    """One scv_ctx bound to one CUDA device."""

    def __init__(self, device: int):
        lib = load_library()
        self.lib = lib
        self.device = device
        self.lock = threading.RLock()
        h = _P()
        rc = lib.scv_create(device, ctypes.byref(h))
        if rc != SCV_OK:
            raise RuntimeError(f"scv_create(device={device}) failed with code {rc}")
        self.handle = h

    def call(self, name: str, *args):
        """Invoke scv_<name>(ctx, *args, stream) on torch's current stream."""
        stream = torch.cuda.current_stream(self.device).cuda_stream
        with self.lock:
            rc = getattr(self.lib, "scv_" + name)(self.handle, *args, _P(stream))
            if rc != SCV_OK:
                msg = self.lib.scv_last_error(self.handle).decode(errors="replace")
                if rc == SCV_EINVAL:
                    raise ValueError(msg)
                if rc == SCV_ETYPE:
                    raise TypeError(msg)
                raise RuntimeError(f"scv_{name} failed ({rc}): {msg}")

    def betaq_restrict(self, L: int, b0: int = 0, nb: int = 0):
        """scv_betaq_restrict: keep only the beta rows [b0, b0+nb) of the quadrature
        table of band limit L on this context (nb = 0 lifts the restriction)."""
        with self.lock:
            rc = self.lib.scv_betaq_restrict(self.handle, int(L), int(b0), int(nb))
            if rc != SCV_OK:
                msg = self.lib.scv_last_error(self.handle).decode(errors="replace")
                if rc == SCV_EINVAL:
                    raise ValueError(msg)
                raise RuntimeError(f"scv_betaq_restrict failed ({rc}): {msg}")

    def launch_count(self) -> int:
        return int(self.lib.scv_launch_count(self.handle))

    def workspace_bytes(self) -> int:
        return int(self.lib.scv_workspace_bytes(self.handle))

    def profile(self, enable: bool):
        with self.lock:
            self.lib.scv_profile(self.handle, 1 if enable else 0)

    def profile_report(self) -> dict:
        """{stage: (count, total_ms)} since the last report (synchronises)."""
        buf = ctypes.create_string_buffer(1 << 16)
        with self.lock:
            rc = self.lib.scv_profile_report(self.handle, buf, len(buf))
        if rc != SCV_OK:
            raise RuntimeError(self.lib.scv_last_error(self.handle).decode())
        out = {}
        for line in buf.value.decode().splitlines():
            name, cnt, ms = line.split()
            out[name] = (int(cnt), float(ms))
        return out

    def fp64_peak_tflops(self) -> float:
        v = ctypes.c_double()
        with self.lock:
            rc = self.lib.scv_fp64_peak(self.handle, ctypes.byref(v))
        if rc != SCV_OK:
            raise RuntimeError(self.lib.scv_last_error(self.handle).decode())
        return v.value

    def dmma_peak_tflops(self) -> float:
        v = ctypes.c_double()
        with self.lock:
            rc = self.lib.scv_dmma_peak(self.handle, ctypes.byref(v))
        if rc != SCV_OK:
            raise RuntimeError(self.lib.scv_last_error(self.handle).decode())
        return v.value

    def set_option(self, name: str, value: int):
        """scv_set_option: e.g. set_option("betaq", 0) selects the FFT beta stage."""
        with self.lock:
            rc = self.lib.scv_set_option(self.handle, name.encode(), int(value))
        if rc != SCV_OK:
            raise ValueError(self.lib.scv_last_error(self.handle).decode())

    def trim(self):
        with self.lock:
            torch.cuda.synchronize(self.device)
            rc = self.lib.scv_trim(self.handle)
        if rc != SCV_OK:
            raise ValueError(self.lib.scv_last_error(self.handle).decode())

    def __del__(self):
        try:
            self.lib.scv_destroy(self.handle)
        except Exception:
            pass


_ctxs: dict = {}
_ctx_lock = threading.Lock()


# A private context (own scratch and tables) bound for the current thread /
# task by `using`, so independent pipelines can run concurrently on separate
# streams without sharing scratch buffers (GraphedRoundTrip lanes).
_override: contextvars.ContextVar = contextvars.ContextVar("scv_context_override", default=None)


def new_context(device: int | None = None) -> Context:
    """A fresh, unshared context on `device` (default: the current device)."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1511_05578_b200 needs a CUDA device (B200); there is no CPU fallback")
    return Context(torch.cuda.current_device() if device is None else int(device))


@contextlib.contextmanager
def using(ctx: Context):
    """Route every library call on ctx's device inside the block to `ctx`."""
    tok = _override.set(ctx)
    try:
        yield ctx
    finally:
        _override.reset(tok)


def context(device: torch.device | int | None = None) -> Context:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1511_05578_b200 needs a CUDA device (B200); there is no CPU fallback")
    if device is None:
        idx = torch.cuda.current_device()
    elif isinstance(device, torch.device):
        idx = device.index if device.index is not None else torch.cuda.current_device()
    else:
        idx = int(device)
    ov = _override.get()
    if ov is not None and ov.device == idx:
        return ov
    with _ctx_lock:
        if idx not in _ctxs:
            _ctxs[idx] = Context(idx)
        return _ctxs[idx]


def ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return _P(t.data_ptr())


def checked(t, dtype: torch.dtype, shape, device, what: str = "buffer") -> torch.Tensor:
    """Validate a caller-supplied tensor before its raw pointer reaches the C
    ABI (which trusts sizes): a CUDA tensor on `device`, exactly `dtype`,
    C-contiguous, exactly `shape`.  TypeError for a non-tensor / wrong dtype,
    ValueError for device, layout or shape mismatches."""
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{what} must be a torch tensor, got {type(t).__name__}")
    if t.dtype != dtype:
        raise TypeError(f"{what} must have dtype {dtype}, got {t.dtype}")
    dev = device if isinstance(device, torch.device) else torch.device("cuda", int(device))
    if not t.is_cuda or (dev.index is not None and t.device.index != dev.index):
        raise ValueError(f"{what} must live on {dev}, got {t.device}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{what} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    return t
