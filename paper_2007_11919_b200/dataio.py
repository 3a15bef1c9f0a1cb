"""File ingestion — the readers of the reference's
``dataio`` module (``src/dataio.py:42-130``) with the same names, arguments
and errors: IDX images streamed straight into device memory (unsigned bytes
over PCIe, widened by a kernel) and numeric CSV parsed by native host
threads.  The reference's writers and run manifest are outside the hot path
and not part of this package.

* ``read_idx_images`` / ``read_idx_labels`` validate the header with the same
  FormatError texts (``dataio.py:42-58, 68-82``); ``IdxImageSet.to_data_matrix``
  is the reference's float64 host matrix, ``IdxImageSet.to_device`` /
  ``load_idx_images`` the device one (bit-identical: u8 -> f64 is exact).
* ``read_csv_matrix`` (``dataio.py:102-130``) runs in ``mdsx_csv_read``:
  correctly rounded like Python ``float()``, same first-error-in-file-order
  messages (ragged row / invalid number / no data rows).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from .errors import FormatError, InvalidInputError

IDX_IMAGES_MAGIC = 0x00000803
IDX_LABELS_MAGIC = 0x00000801


def _probe(path, kind: int) -> tuple[int, int, int]:
    os.stat(path)                                  # FileNotFoundError like Path.read_bytes()
    lib = _lib.load()
    n, h, w = C.c_int64(), C.c_int32(), C.c_int32()
    msg = C.create_string_buffer(1024)
    rc = lib.mdsx_idx_probe(os.fsencode(str(path)), kind, C.byref(n), C.byref(h), C.byref(w),
                            msg, len(msg))
    if rc != _lib.OK:
        raise _lib.status_error(rc, msg.value.decode(errors="replace"))
    return n.value, h.value, w.value


@dataclass(frozen=True)
class IdxImageSet:
    """A stack of equally sized grayscale images, pixel values 0-255."""

    height: int
    width: int
    pixels: np.ndarray  # (count, height, width) uint8
    path: str | None = None

    @property
    def count(self) -> int:
        return self.pixels.shape[0]

    def to_data_matrix(self) -> np.ndarray:
        """Flatten row-major into a (count, height*width) float64 matrix (host)."""
        return self.pixels.reshape(self.count, self.height * self.width).astype(np.float64)

    def to_device(self, device=None, dtype=None, scale: float = 1.0):
        """The same matrix on the device (u8 over PCIe, widened by a kernel);
        from the file when this set was read from one."""
        if self.path is not None:
            return load_idx_images(self.path, device=device, dtype=dtype, scale=scale)
        import torch
        from . import _device as D
        dev = D.require_device(device)
        dt = dtype or torch.float64
        u8 = torch.from_numpy(np.ascontiguousarray(self.pixels)).to(dev)
        return (u8.reshape(self.count, -1).to(dt) * scale) if scale != 1.0 else \
            u8.reshape(self.count, -1).to(dt)


def read_idx_images(path) -> IdxImageSet:
    """Parse an IDX image file (magic 0x00000803)."""
    n, h, w = _probe(path, 3)
    pixels = np.fromfile(str(path), dtype=np.uint8, offset=16).reshape(n, h, w)
    return IdxImageSet(height=h, width=w, pixels=pixels, path=str(path))


def load_idx_images(path, *, device=None, dtype=None, scale: float = 1.0):
    """IDX images -> device matrix (count x height*width) of ``dtype`` (torch
    float64 by default), element = scale * pixel.  The file is streamed in
    32 MB chunks through pinned buffers; only the unsigned bytes cross PCIe."""
    import torch
    from . import _device as D
    n, h, w = _probe(path, 3)
    dev = D.require_device(device)
    dt = dtype or torch.float64
    if dt not in (torch.float64, torch.float32):
        raise ValueError("dtype must be torch.float64 or torch.float32")
    out = torch.empty((n, h * w), dtype=dt, device=dev)
    code = _lib.F64 if dt == torch.float64 else _lib.F32
    D.handle(dev).call("mdsx_idx_load_images", os.fsencode(str(path)), out.data_ptr(), code,
                       float(scale), D.stream_ptr(dev))
    return out


def read_idx_labels(path) -> np.ndarray:
    """Parse an IDX label file (magic 0x00000801) into a uint8 vector."""
    n, _, _ = _probe(path, 1)
    return np.fromfile(str(path), dtype=np.uint8, offset=8).copy()


def read_csv_matrix(path, has_header: bool = False, *, threads: int = 0) -> np.ndarray:
    """Read a rectangular numeric CSV into a float64 matrix (native parser).

    Ragged or non-numeric rows raise FormatError naming the line number
    (1-based, counting the header if present); ``threads`` = 0 uses every core.
    """
    os.stat(path)                                  # FileNotFoundError like open()
    lib = _lib.load()
    p = os.fsencode(str(path))
    rows, cols = C.c_int64(), C.c_int64()
    msg = C.create_string_buffer(1024)
    rc = lib.mdsx_csv_read(p, int(bool(has_header)), int(threads), None, C.byref(rows),
                           C.byref(cols), msg, len(msg))
    if rc != _lib.OK:
        raise _lib.status_error(rc, msg.value.decode(errors="replace"))
    out = np.empty((rows.value, cols.value), dtype=np.float64)
    buf = out if out.size else np.empty(1, dtype=np.float64)
    rc = lib.mdsx_csv_read(p, int(bool(has_header)), int(threads), buf.ctypes.data,
                           C.byref(rows), C.byref(cols), msg, len(msg))
    if rc != _lib.OK:
        raise _lib.status_error(rc, msg.value.decode(errors="replace"))
    return out
