"""Device plumbing shared by the host API: CUDA checks, streams, error words,
host<->device staging.  PyTorch is used only for device memory and streams."""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

_TORCH_CODE = {torch.bfloat16: _lib.BF16, torch.float32: _lib.F32, torch.float64: _lib.F64}
_INTLOG_LOADED: set[tuple[int, int]] = set()


def require_cuda() -> torch.device:
    """The product path has no CPU fallback: fail loudly without a GPU."""
    _lib.lib()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2508_03760_b200 needs a CUDA device (B200, sm_100a); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _TORCH_CODE[t.dtype]
    except KeyError as exc:
        raise TypeError(f"unsupported element type {t.dtype}; use bf16, float32 or float64") from exc


def is_cuda_tensor(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def to_device_values(values, device) -> torch.Tensor:
    """Stage a host array for the encoder without changing its value set:
    float16/float32 travel as float32 (exact), everything else as float64
    (the reference widens to float64, codec.py:479)."""
    if isinstance(values, torch.Tensor):
        t = values.detach()
        if t.dtype not in _TORCH_CODE:
            t = t.to(torch.float64)
        return t.to(device, non_blocking=False).contiguous()
    arr = np.asarray(values)
    if arr.dtype in (np.float32, np.float16):
        arr = arr.astype(np.float32, copy=False)
    else:
        arr = np.asarray(values, dtype=np.float64)
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device)


def new_err(device) -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=device)


def check_err(err: torch.Tensor, what: str = "") -> None:
    bits = int(err.item())
    if bits:
        _lib.raise_dev_err(bits, what)


def ensure_intlog(theta: int, device) -> None:
    """Upload exp2(si/theta), si=-128..127, computed by numpy exactly as the
    reference does (codec.py:468,542) so device scales are bit-identical."""
    key = (int(theta), device.index if device.index is not None else torch.cuda.current_device())
    if key in _INTLOG_LOADED:
        return
    table = np.exp2(np.arange(-128, 128, dtype=np.float64) / theta)
    buf = np.ascontiguousarray(table, dtype=np.float64)
    with torch.cuda.device(key[1]):
        _lib.check(_lib.lib().fc2_set_intlog_table(int(theta), buf.ctypes.data_as(
            __import__("ctypes").POINTER(__import__("ctypes").c_double))))
    _INTLOG_LOADED.add(key)


_WORKSPACES: dict[tuple[int, str], torch.Tensor] = {}


def workspace(name: str, nbytes: int, device) -> torch.Tensor:
    """A cached uint8 device buffer of at least ``nbytes`` (staging for the
    host-resident pipeline; grown, never shrunk)."""
    idx = device.index if device.index is not None else torch.cuda.current_device()
    key = (idx, name)
    buf = _WORKSPACES.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=torch.device("cuda", idx))
        _WORKSPACES[key] = buf
    return buf
