"""Device plumbing: input coercion/staging, streams, small D2H reads.

PyTorch is used only for device memory, streams and copies."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import InvalidInputError


def require_device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("a CUDA device is required: this package has no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise RuntimeError(f"device {dev} is not a CUDA device (no CPU fallback)")
    return torch.device("cuda", dev.index if dev.index is not None else torch.cuda.current_device())


def stream_ptr(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def handle(dev: torch.device) -> _lib.Handle:
    return _lib.Handle.get(dev.index)


def dtype_code(t: torch.Tensor) -> int:
    return _lib.F32 if t.dtype == torch.float32 else _lib.F64


def host_matrix(data, name: str = "data") -> np.ndarray:
    """Shape checks of linalg.py:28-38 on the host (finiteness is checked by
    the kernels that read the data).  float32 stays float32 (read and widened
    to float64 on the device); anything else becomes float64."""
    if isinstance(data, np.ndarray) and data.dtype in (np.float32, np.float64):
        arr = data
    else:
        arr = np.asarray(data, dtype=np.float64)
    if arr.ndim != 2:
        raise InvalidInputError(f"{name} must be 2-dimensional, got ndim={arr.ndim}")
    if arr.shape[0] < 1 or arr.shape[1] < 1:
        raise InvalidInputError(f"{name} must be non-empty, got shape {arr.shape}")
    return arr


def to_device_matrix(data, dev: torch.device, name: str = "data") -> torch.Tensor:
    """Device-resident row-major float32/float64 matrix for the C-ABI."""
    if isinstance(data, torch.Tensor):
        t = data
        if t.dim() != 2:
            raise InvalidInputError(f"{name} must be 2-dimensional, got ndim={t.dim()}")
        if t.shape[0] < 1 or t.shape[1] < 1:
            raise InvalidInputError(f"{name} must be non-empty, got shape {tuple(t.shape)}")
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        if t.device != dev:
            t = t.to(dev, non_blocking=t.device.type == "cpu" and t.is_pinned())
        return t.contiguous()
    arr = np.ascontiguousarray(host_matrix(data, name))
    return from_host(arr, dev)


def from_host(arr: np.ndarray, dev: torch.device) -> torch.Tensor:
    """Device copy of a host array.  Large pageable arrays go through the
    library's staged copy (mdsx_h2d: page-locked chunk buffers filled by
    several host threads while earlier chunks are in flight over PCIe); a
    plain pageable copy runs at a few GB/s on the B200 hosts."""
    t = torch.from_numpy(arr)
    if arr.nbytes < (4 << 20):
        return t.to(dev)
    out = torch.empty(t.shape, dtype=t.dtype, device=dev)
    handle(dev).call("mdsx_h2d", out.data_ptr(), arr.ctypes.data, arr.nbytes, 0, stream_ptr(dev))
    return out


COMPACT_MIN_P = 105          # the block-Krylov shapes (k > 104); narrower inputs skip the pass
COMPACT_MAX_ACTIVE = 0.9     # compact when at most this fraction of the columns is active


class ColumnCompactor:
    """Column compaction of a wide device matrix (k_compact.cu): at every call
    one pass finds the columns with a nonzero entry (the data may change
    between launches), and when at most 90% are active they are gathered into
    a persistent dense buffer whose rows stay 16-byte multiples; the
    algorithms then run on it and return the same configuration (zero columns
    contribute exactly zero to every Gram, eigenvector, mean, point and Gower
    term).  Narrow inputs are returned as they are."""

    def __init__(self, x: torch.Tensor):
        self.x = x
        self.buf = None
        self.active = None           # number of active columns of the last call

    def __call__(self) -> torch.Tensor:
        import ctypes as C
        x = self.x
        n, p = x.shape
        if p < COMPACT_MIN_P:
            return x
        dev = x.device
        h = handle(dev)
        cols = np.empty(p, dtype=np.int32)
        cnt = C.c_int32(0)
        h.call("mdsx_active_columns", x.data_ptr(), dtype_code(x), x.stride(0), n, p,
               cols.ctypes.data, C.byref(cnt), stream_ptr(dev))
        pa = self.active = int(cnt.value)
        if pa == 0 or pa > COMPACT_MAX_ACTIVE * p:
            return x
        vw = 16 // x.element_size()
        ldo = -(-pa // vw) * vw
        if self.buf is None or tuple(self.buf.shape) != (n, ldo):
            self.buf = torch.empty((n, ldo), dtype=x.dtype, device=dev)
        cols_dev = torch.from_numpy(cols[:pa].copy()).to(dev)
        h.call("mdsx_gather_columns", x.data_ptr(), dtype_code(x), x.stride(0), n,
               cols_dev.data_ptr(), pa, ldo, self.buf.data_ptr(), stream_ptr(dev))
        return self.buf


def index_tensor(idx: np.ndarray, dev: torch.device) -> torch.Tensor:
    """Upload an int64 index array.  Large arrays go through page-locked
    staging and an async copy (stream-ordered; torch's caching host allocator
    keeps the staging block alive until the copy has completed)."""
    a = np.ascontiguousarray(idx, dtype=np.int64)
    if a.nbytes < (1 << 20):
        return torch.from_numpy(a).to(dev)
    pin = torch.empty(a.shape, dtype=torch.int64, pin_memory=True)
    pin.numpy()[...] = a
    return pin.to(dev, non_blocking=True)


def empty(shape, dev: torch.device, dtype=torch.float64) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=dev)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


STATUS_DTYPE = np.dtype([("code", np.int32), ("index", np.int32), ("value", np.float64)])


def status_tensor(n: int, dev: torch.device) -> torch.Tensor:
    return torch.zeros((n, 2), dtype=torch.float64, device=dev)  # 16 B per record


def decode_status(t: torch.Tensor) -> np.ndarray:
    raw = t.detach().cpu().numpy().view(np.uint8).reshape(-1, 16)
    return raw.copy().view(STATUS_DTYPE).reshape(-1)


def to_host(t: torch.Tensor) -> np.ndarray:
    """D2H through page-locked memory (torch's caching host allocator): pageable
    copies of large results run at a few GB/s on the B200 hosts, pinned at
    PCIe speed.  The returned array owns its pinned block until collected."""
    if not t.is_cuda:
        return t.numpy()
    pin = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    pin.copy_(t)
    return pin.numpy()
