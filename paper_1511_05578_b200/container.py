"""SCRV1 coefficient containers, streamed between HBM and disk.

Byte-compatible mirror of the reference's ``scurve.container`` writers and
readers (container.py:58-236): the 5-byte magic ``SCRV1``, a little-endian
uint32 header length, the UTF-8 JSON header with the same keys in the same
order and the same section table, then the raw little-endian payload
sections.  A file written here is byte-identical to the reference's for the
same values (tests/test_container.py checks it against reference-written
fixtures).

What changes is the data path.  A C4 map is 147 GB of coefficients, so
nothing is materialised on the host.  The writer streams every device section
through two pinned staging buffers. The D2H copy of chunk i+1 runs on a side
stream while chunk i is written to the file. The reader validates the whole
section table against the file size first, as the reference does. It then
streams each section from disk into pinned buffers and H2D into its
preallocated device tensor, with the same overlap.  Writes keep the
reference's atomic semantics: a temporary file next to the target, fsync,
then rename.  PGM ingest and resampling (container.py:239-300) are image UX
outside the transform path and stay out of scope.
"""

from __future__ import annotations

import json
import os
import struct
import tempfile

import numpy as np
import torch

from .so3 import SO3Grid, SO3Signal
from .sphere import SphereGrid, SphereSignal
from .tiling import TilingParams
from .transform import CurveletCoeffs, scale_band_limit, scaling_band_limit

__all__ = [
    "MAGIC",
    "ContainerError",
    "read_coeffs",
    "read_container",
    "read_sphere",
    "write_coeffs",
    "write_sphere",
]

MAGIC = b"SCRV1"

_HEADER_CAP = 1 << 24
_DTYPES = {"<f8": np.dtype("<f8"), "<c16": np.dtype("<c16")}
_TORCH = {"<f8": torch.float64, "<c16": torch.complex128}
_RESERVED = frozenset(("kind", "L", "spin", "lambda", "J0", "J", "frame", "multires", "real", "sections"))
CHUNK_BYTES = 64 << 20  # pinned staging buffer size (two of them per transfer)


class ContainerError(RuntimeError):
    """Malformed, truncated or inconsistent container data."""


def _is_complex(v) -> bool:
    return v.is_complex() if isinstance(v, torch.Tensor) else np.iscomplexobj(v)


def _payload_code(values) -> str:
    return "<c16" if _is_complex(values) else "<f8"


def _merge_extra(header: dict, extra) -> None:
    if not extra:
        return
    clash = sorted(set(extra) & _RESERVED)
    if clash:
        raise ValueError(f"extra header keys collide with reserved names: {clash}")
    header.update(extra)


def _as_bytes_view(v) -> tuple:
    """(flat byte view, on_device) of a section array without copying to host."""
    if isinstance(v, torch.Tensor):
        t = v.detach()
        t = t.to(_TORCH[_payload_code(t)]).contiguous().reshape(-1)
        if t.is_complex():
            t = torch.view_as_real(t).reshape(-1)
        return t.view(torch.uint8), t.is_cuda
    a = np.ascontiguousarray(v, dtype=_DTYPES[_payload_code(v)])
    return a.reshape(-1).view(np.uint8), False


class _Stager:
    """Two pinned host buffers and a side stream for overlapped HBM <-> disk transfers."""

    def __init__(self, device: torch.device, chunk: int):
        self.chunk = chunk
        self.stream = torch.cuda.Stream(device)
        self.bufs = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        self.events = [torch.cuda.Event(), torch.cuda.Event()]
        self.busy = [False, False]

    def drain(self, i):
        if self.busy[i]:
            self.events[i].synchronize()
            self.busy[i] = False

    def d2h(self, fh, src: torch.Tensor) -> None:
        """Write the device bytes `src` to fh: D2H of chunk i+1 overlaps the write of chunk i."""
        self.stream.wait_stream(torch.cuda.current_stream(src.device))
        n, off, i, pending = src.numel(), 0, 0, None
        while off < n:
            k = min(self.chunk, n - off)
            b = self.bufs[i & 1]
            with torch.cuda.stream(self.stream):
                b[:k].copy_(src[off: off + k], non_blocking=True)
                self.events[i & 1].record(self.stream)
            if pending is not None:
                j, kk = pending
                self.events[j].synchronize()
                fh.write(memoryview(self.bufs[j][:kk].numpy()))
            pending, off, i = (i & 1, k), off + k, i + 1
        if pending is not None:
            j, kk = pending
            self.events[j].synchronize()
            fh.write(memoryview(self.bufs[j][:kk].numpy()))
        src.record_stream(self.stream)

    def h2d(self, fh, dst: torch.Tensor, path) -> None:
        """Fill the device bytes `dst` from fh: the read of chunk i+1 overlaps the H2D of chunk i."""
        n, off, i = dst.numel(), 0, 0
        while off < n:
            k = min(self.chunk, n - off)
            j = i & 1
            self.drain(j)  # buffer j's previous H2D must have finished
            view = memoryview(self.bufs[j][:k].numpy())
            got = fh.readinto(view)
            if got != k:
                raise ContainerError(f"{path}: payload truncated while reading")
            with torch.cuda.stream(self.stream):
                dst[off: off + k].copy_(self.bufs[j][:k], non_blocking=True)
                self.events[j].record(self.stream)
            self.busy[j] = True
            off, i = off + k, i + 1
        self.drain(0)
        self.drain(1)
        dst.record_stream(self.stream)


def _write_container(path, header: dict, arrays, chunk: int = CHUNK_BYTES) -> None:
    """arrays is a list of (name, tensor | ndarray); the section table is derived
    from shapes and dtypes alone, so the header is written before any payload."""
    sections, views = [], []
    offset = 0
    for name, arr in arrays:
        code = _payload_code(arr)
        view, on_dev = _as_bytes_view(arr)
        nbytes = int(view.numel() if on_dev or isinstance(view, torch.Tensor) else view.size)
        sections.append({"name": name, "dtype": code, "shape": [int(d) for d in arr.shape],
                         "offset": offset, "nbytes": nbytes})
        views.append((view, on_dev))
        offset += nbytes
    head = json.dumps(dict(header, sections=sections), allow_nan=False).encode()
    directory = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(dir=directory, prefix=".scrv-")
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(MAGIC)
            fh.write(struct.pack("<I", len(head)))
            fh.write(head)
            stager = None
            for view, on_dev in views:
                if on_dev:
                    if stager is None:
                        stager = _Stager(view.device, chunk)
                    stager.d2h(fh, view)
                elif isinstance(view, torch.Tensor):
                    fh.write(memoryview(view.numpy()))
                else:
                    fh.write(memoryview(view))
            fh.flush()
            os.fsync(fh.fileno())
        os.replace(tmp, path)
    except BaseException:
        try:
            os.unlink(tmp)
        except OSError:
            pass
        raise


def _read_layout(path, fh, size: int):
    """Parse and validate the header and section table (container.py:111-149)."""
    pre = fh.read(len(MAGIC) + 4)
    if len(pre) < len(MAGIC) + 4 or pre[: len(MAGIC)] != MAGIC:
        raise ContainerError(f"{path}: not an SCRV1 container")
    (hlen,) = struct.unpack_from("<I", pre, len(MAGIC))
    start = len(MAGIC) + 4
    if hlen > _HEADER_CAP or start + hlen > size:
        raise ContainerError(f"{path}: header length {hlen} exceeds file size")
    try:
        header = json.loads(fh.read(hlen).decode())
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise ContainerError(f"{path}: bad header: {exc}") from None
    if not isinstance(header, dict) or not isinstance(header.get("sections"), list):
        raise ContainerError(f"{path}: header carries no section table")
    payload = size - start - hlen
    layout = []
    seen = set()
    for sec in header["sections"]:
        try:
            name = sec["name"]
            code = sec["dtype"]
            shape = tuple(int(d) for d in sec["shape"])
            offset = int(sec["offset"])
            nbytes = int(sec["nbytes"])
        except (TypeError, KeyError, ValueError) as exc:
            raise ContainerError(f"{path}: malformed section entry: {exc}") from None
        if name in seen:
            raise ContainerError(f"{path}: duplicate section {name!r}")
        seen.add(name)
        if code not in _DTYPES:
            raise ContainerError(f"{path}: unknown payload dtype {code!r}")
        count = int(np.prod(shape, dtype=np.int64))
        if nbytes != count * _DTYPES[code].itemsize:
            raise ContainerError(f"{path}: section {name!r} length does not match its shape")
        if offset < 0 or offset + nbytes > payload:
            raise ContainerError(f"{path}: section {name!r} exceeds the payload")
        layout.append((name, code, shape, start + hlen + offset, nbytes))
    return header, layout


def read_container(path, device=None, chunk: int = CHUNK_BYTES):
    """Return (header, {section name: tensor}) after validating the layout.

    Sections land on `device` (default: the current CUDA device); with
    device="cpu" they are host tensors read directly from the file."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    size = os.path.getsize(path)
    out = {}
    with open(path, "rb", buffering=0) as fh:
        header, layout = _read_layout(path, fh, size)
        stager = None
        for name, code, shape, pos, nbytes in layout:
            t = torch.empty(shape, dtype=_TORCH[code], device=dev)
            flat = t.reshape(-1)
            if t.is_complex():
                flat = torch.view_as_real(flat).reshape(-1)
            raw = flat.view(torch.uint8)
            fh.seek(pos)
            if dev.type == "cuda":
                if stager is None:
                    stager = _Stager(dev, chunk)
                stager.h2d(fh, raw, path)
            else:
                if fh.readinto(memoryview(raw.numpy())) != nbytes:
                    raise ContainerError(f"{path}: payload truncated while reading")
            out[name] = t
    return header, out


def write_sphere(path, signal: SphereSignal, extra=None) -> None:
    """Write one sphere signal; extra adds provenance keys (container.py:152-166)."""
    header = {"kind": "sphere", "L": signal.grid.band_limit, "spin": signal.spin, "lambda": None,
              "J0": None, "J": None, "frame": None, "multires": None, "real": signal.real}
    _merge_extra(header, extra)
    _write_container(path, header, [("values", signal.values)])


def read_sphere(path) -> SphereSignal:
    """container.py:169-185, onto the current CUDA device."""
    header, sections = read_container(path)
    if header.get("kind") != "sphere":
        raise ContainerError(f"{path}: not a sphere container")
    try:
        L = int(header["L"])
        spin = int(header["spin"])
        real = bool(header["real"])
        values = sections["values"]
    except (KeyError, TypeError, ValueError) as exc:
        raise ContainerError(f"{path}: incomplete sphere header: {exc}") from None
    if real and values.is_complex():
        raise ContainerError(f"{path}: real-flagged payload stored as complex")
    try:
        return SphereSignal(SphereGrid(L), spin, values, real=real)
    except ValueError as exc:
        raise ContainerError(f"{path}: {exc}") from None


def _coeff_header(p: TilingParams, frame, multires, real, extra) -> dict:
    header = {"kind": "curvelet", "L": p.band_limit, "spin": p.spin, "lambda": p.lam, "J0": p.j_min,
              "J": p.j_max, "frame": frame, "multires": multires, "real": real}
    _merge_extra(header, extra)
    return header


def write_coeffs(path, coeffs: CurveletCoeffs, extra=None) -> None:
    """Write an analysis result: the scaling part plus every scale signal
    (container.py:188-206), streamed section by section from HBM."""
    p = coeffs.params
    header = _coeff_header(p, coeffs.frame, coeffs.multires, coeffs.real, extra)
    arrays = [("scaling", coeffs.scaling.values)]
    for j in range(p.j_min, p.j_max + 1):
        arrays.append((f"scale_{j}", coeffs.scale(j).values))
    _write_container(path, header, arrays)


def read_coeffs(path) -> CurveletCoeffs:
    """container.py:209-236, each section streamed straight into HBM."""
    header, sections = read_container(path)
    if header.get("kind") != "curvelet":
        raise ContainerError(f"{path}: not a curvelet-coefficient container")
    try:
        params = TilingParams(int(header["L"]), int(header["spin"]), float(header["lambda"]),
                              int(header["J0"]), int(header["J"]))
        frame = header["frame"]
        multires = bool(header["multires"])
        real = bool(header["real"])
    except (KeyError, TypeError, ValueError) as exc:
        raise ContainerError(f"{path}: incomplete coefficient header: {exc}") from None
    L = params.band_limit
    try:
        low = scaling_band_limit(params) if multires else L
        scaling = SphereSignal(SphereGrid(low), 0, sections["scaling"], real=real)
        scales = []
        for j in range(params.j_min, params.j_max + 1):
            Lj = scale_band_limit(params, j) if multires else L
            scales.append(SO3Signal(SO3Grid(Lj, Lj, Lj), sections[f"scale_{j}"], real=real))
        return CurveletCoeffs(params, frame, scaling, scales, multires, real)
    except (KeyError, ValueError) as exc:
        raise ContainerError(f"{path}: {exc}") from None
