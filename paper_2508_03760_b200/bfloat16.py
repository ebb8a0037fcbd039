"""bfloat16 helpers (reference: bfloat16.py:16-41) computed on the GPU.

Host arrays round-trip through the device; CUDA tensors stay there.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device, _lib


def _f32_device(x):
    dev = _device.require_cuda()
    if _device.is_cuda_tensor(x):
        return x.detach().reshape(-1).to(torch.float32).contiguous(), True, tuple(x.shape)
    arr = np.asarray(x, dtype=np.float32)
    return torch.from_numpy(np.ascontiguousarray(arr).reshape(-1)).to(dev), False, arr.shape


def f32_to_bf16_bits(x):
    """float32 -> bf16 bit patterns, round-to-nearest-even (bfloat16.py:16-25)."""
    t, dev_in, shape = _f32_device(x)
    out = torch.empty(t.numel(), dtype=torch.int16, device=t.device)
    _lib.check(_lib.lib().fc2_f32_to_bf16_bits(t.data_ptr(), t.numel(), out.data_ptr(),
                                               _device.stream_handle()))
    if dev_in:
        return out.view(torch.uint16).reshape(shape) if hasattr(torch, "uint16") else out.reshape(shape)
    return out.cpu().numpy().view(np.uint16).reshape(shape)


def bf16_bits_to_f32(bits):
    """Widen bf16 bit patterns to float32, exactly (bfloat16.py:28-31)."""
    dev = _device.require_cuda()
    if _device.is_cuda_tensor(bits):
        t = bits.detach().reshape(-1).view(torch.int16).contiguous()
        dev_in, shape = True, tuple(bits.shape)
    else:
        arr = np.asarray(bits, dtype=np.uint16)
        t = torch.from_numpy(np.ascontiguousarray(arr).reshape(-1).view(np.int16)).to(dev)
        dev_in, shape = False, arr.shape
    out = torch.empty(t.numel(), dtype=torch.float32, device=t.device)
    _lib.check(_lib.lib().fc2_bf16_bits_to_f32(t.data_ptr(), t.numel(), out.data_ptr(),
                                               _device.stream_handle()))
    if dev_in:
        return out.reshape(shape)
    return out.cpu().numpy().reshape(shape)


def bf16_round(x):
    """Snap to the bf16 grid, returned as float32 (bfloat16.py:34-36)."""
    return bf16_bits_to_f32(f32_to_bf16_bits(x))


def bf16_round_scalar(x: float) -> float:
    return float(np.asarray(bf16_round(np.float32(x))).reshape(()))
