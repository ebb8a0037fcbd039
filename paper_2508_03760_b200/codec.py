"""Drop-in codec API (reference: codec.py) on the B200 CUDA library.

``encode_chunk`` / ``decode_chunk`` / ``pack_codes`` / ``unpack_codes`` keep
the reference names, argument meaning and exceptions.  All arithmetic runs in
libfc2.so on the GPU; host code only validates shapes and moves bytes.

Two residencies:
* host in, host out (the reference contract): numpy/list input, the returned
  :class:`QuantizedChunk` holds ``bytes``; ``decode_chunk`` returns float64
  numpy bit-identical to the reference.
* device resident: a CUDA tensor input keeps the payload on the GPU
  (``chunk.payload``); ``decode_chunk`` then returns a CUDA tensor
  (float32 unless ``out_dtype`` says otherwise).
"""

from __future__ import annotations

import ctypes
import struct

import numpy as np
import torch

from . import _device, _lib
from .config import (
    GroupMeta,
    QuantConfig,
    ScaleEncoding,
    Scheme,
    bit_split,
    default_group_size,
    footprint_breakdown,
    footprint_bytes,
    meta_record_nbytes,
    plane_sizes,
)
from .errors import ConfigError, DataError, DecodeFormatError

CHUNK_MAGIC = b"FCV2"
CHUNK_VERSION = 2
_HEADER = struct.Struct("<4sBBHBBBI")  # codec.py:33-35
HEADER_BYTES = _HEADER.size

__all__ = [
    "QuantConfig", "Scheme", "ScaleEncoding", "GroupMeta", "QuantizedChunk",
    "bit_split", "default_group_size", "footprint_bytes", "footprint_breakdown",
    "meta_record_nbytes", "encode_chunk", "decode_chunk", "pack_codes", "unpack_codes",
    "parse_chunk", "encode_payload", "decode_payload", "encode_host", "decode_host", "roundtrip_host",
]


class QuantizedChunk:
    """Packed code planes + per-group metadata (codec.py:105-136).

    Host chunks hold ``bytes``; device chunks hold one contiguous uint8 CUDA
    tensor ``payload`` (planes in split order, then metadata) and materialize
    ``planes``/``meta`` bytes lazily.
    """

    def __init__(self, config: QuantConfig, planes=None, meta=None, element_count: int = 0,
                 *, payload: torch.Tensor | None = None):
        self.config = config
        self.element_count = int(element_count)
        self._payload = payload
        self._planes = None if planes is None else [bytes(p) for p in planes]
        self._meta = None if meta is None else bytes(meta)
        if payload is None and (self._planes is None or self._meta is None):
            raise DataError("QuantizedChunk needs planes and meta, or a device payload")

    # -- residency ---------------------------------------------------------
    @property
    def on_device(self) -> bool:
        return self._payload is not None

    @property
    def payload(self) -> torch.Tensor:
        """The payload as one uint8 CUDA tensor (uploads host bytes once)."""
        if self._payload is None:
            dev = _device.require_cuda()
            buf = np.frombuffer(b"".join(self._planes) + self._meta, dtype=np.uint8)
            self._payload = torch.from_numpy(buf.copy()).to(dev)
        return self._payload

    def _materialize(self):
        raw = self._payload.cpu().numpy().tobytes()
        sizes = plane_sizes(self.config, self.element_count)
        planes, pos = [], 0
        for s in sizes:
            planes.append(raw[pos:pos + s])
            pos += s
        self._planes, self._meta = planes, raw[pos:]

    @property
    def planes(self) -> list[bytes]:
        if self._planes is None:
            self._materialize()
        return self._planes

    @property
    def meta(self) -> bytes:
        if self._meta is None:
            self._materialize()
        return self._meta

    @property
    def payload_nbytes(self) -> int:
        if self._payload is not None:
            return int(self._payload.numel())
        return sum(len(p) for p in self._planes) + len(self._meta)

    # -- wire format (host framing, codec.py:118-136) ------------------------
    def to_bytes(self) -> bytes:
        c = self.config
        header = _HEADER.pack(CHUNK_MAGIC, CHUNK_VERSION, c.bitwidth, c.group_size,
                              0 if c.scheme is Scheme.RTN else 1,
                              0 if c.scale_encoding is ScaleEncoding.BF16 else 1,
                              c.theta, self.element_count)
        return header + b"".join(self.planes) + self.meta

    @classmethod
    def from_bytes(cls, buf: bytes) -> "QuantizedChunk":
        chunk, consumed = parse_chunk(buf, 0)
        if consumed != len(buf):
            raise DecodeFormatError(f"{len(buf) - consumed} trailing bytes after chunk")
        return chunk

    def __eq__(self, other):
        if not isinstance(other, QuantizedChunk):
            return NotImplemented
        return (self.config == other.config and self.element_count == other.element_count
                and self.planes == other.planes and self.meta == other.meta)

    def __repr__(self):
        where = "device" if self.on_device else "host"
        return (f"QuantizedChunk(bits={self.config.bitwidth}, g={self.config.group_size}, "
                f"scheme={self.config.scheme.value}, n={self.element_count}, "
                f"bytes={self.payload_nbytes}, {where})")


def parse_chunk(buf: bytes, offset: int = 0) -> tuple[QuantizedChunk, int]:
    """Parse one serialized chunk at ``offset``; returns (chunk, end) (codec.py:566-606)."""
    if len(buf) - offset < HEADER_BYTES:
        raise DecodeFormatError("buffer too short for chunk header")
    magic, version, bits, gs, sch, enc, theta, count = _HEADER.unpack_from(buf, offset)
    if magic != CHUNK_MAGIC:
        raise DecodeFormatError(f"bad magic {magic!r}")
    if version != CHUNK_VERSION:
        raise DecodeFormatError(f"unsupported version {version}")
    if sch not in (0, 1) or enc not in (0, 1):
        raise DecodeFormatError("unknown scheme or scale-encoding byte")
    try:
        config = QuantConfig(bits, group_size=gs,
                             scheme=Scheme.RTN if sch == 0 else Scheme.SPIKE_RESERVING,
                             scale_encoding=ScaleEncoding.BF16 if enc == 0 else ScaleEncoding.INT_LOG,
                             theta=theta, chunk_size=count if count > 0 else gs)
    except ConfigError as exc:
        raise DecodeFormatError(f"inconsistent chunk header: {exc}") from exc
    if count % gs:
        raise DecodeFormatError(f"element count {count} not a multiple of group size {gs}")
    pos = offset + HEADER_BYTES
    planes = []
    for w in bit_split(bits):
        size = count * w // 8
        if len(buf) - pos < size:
            raise DecodeFormatError("buffer truncated inside code planes")
        planes.append(bytes(buf[pos:pos + size]))
        pos += size
    msize = (count // gs) * meta_record_nbytes(config)
    if len(buf) - pos < msize:
        raise DecodeFormatError("buffer truncated inside metadata")
    meta = bytes(buf[pos:pos + msize])
    return QuantizedChunk(config, planes, meta, count), pos + msize


# ---------------------------------------------------------------------------
# device-level entry points (tensors in, tensors out; no host sync unless checked)
# ---------------------------------------------------------------------------


def encode_payload(x: torch.Tensor, config: QuantConfig, n: int | None = None,
                   out: torch.Tensor | None = None, err: torch.Tensor | None = None,
                   check: bool = True) -> torch.Tensor:
    """Encode a 1-D CUDA tensor (bf16/f32/f64) as one chunk of ``n`` elements
    (``n >= x.numel()``, zero-padded) into a uint8 CUDA payload."""
    dev = _device.require_cuda()
    if config.int_log:
        _device.ensure_intlog(config.theta, dev)
    x = x.reshape(-1)
    nv = x.numel()
    n = nv if n is None else int(n)
    nbytes = footprint_bytes(config, n)
    if n < nv:
        raise ConfigError(f"chunk of {n} elements cannot hold {nv} values")
    if out is None:
        out = torch.empty(nbytes, dtype=torch.uint8, device=x.device)
    elif (out.device != x.device or out.dtype != torch.uint8 or not out.is_contiguous()
          or out.numel() < nbytes):
        raise ConfigError(f"payload buffer must be a contiguous uint8 tensor of >= {nbytes} bytes on {x.device}")
    own_err = err is None
    if own_err:
        err = _device.new_err(x.device)
    cfg = config.c_struct()
    _lib.check(_lib.lib().fc2_encode(ctypes.byref(cfg), x.data_ptr(), _device.dtype_code(x), nv, n,
                                     out.data_ptr(), err.data_ptr(), _device.stream_handle()))
    if check and own_err:
        _device.check_err(err)
    return out


def decode_payload(payload: torch.Tensor, config: QuantConfig, n: int,
                   out_dtype: torch.dtype = torch.float32, n_out: int | None = None,
                   out: torch.Tensor | None = None, err: torch.Tensor | None = None,
                   check: bool = True) -> torch.Tensor:
    """Decode a uint8 CUDA payload of ``n`` elements into ``out_dtype``
    (bf16 / float32 / float64), keeping the first ``n_out`` values."""
    dev = _device.require_cuda()
    if config.int_log:
        _device.ensure_intlog(config.theta, dev)
    n_out = n if n_out is None else int(n_out)
    need = footprint_bytes(config, n)
    if payload.dtype != torch.uint8 or not payload.is_contiguous() or payload.numel() < need:
        raise ConfigError(f"payload must be a contiguous uint8 tensor of >= {need} bytes")
    if n_out > n:
        raise ConfigError(f"n_out {n_out} exceeds the chunk's {n} elements")
    if out is None:
        out = torch.empty(n_out, dtype=out_dtype, device=payload.device)
    elif out.device != payload.device or not out.is_contiguous() or out.numel() < n_out:
        raise ConfigError(f"out must be a contiguous tensor of >= {n_out} elements on {payload.device}")
    own_err = err is None
    if own_err:
        err = _device.new_err(payload.device)
    cfg = config.c_struct()
    _lib.check(_lib.lib().fc2_decode(ctypes.byref(cfg), payload.data_ptr(), n, out.data_ptr(),
                                     _device.dtype_code(out), n_out, err.data_ptr(),
                                     _device.stream_handle()))
    if check and own_err:
        _device.check_err(err)
    return out


# ---------------------------------------------------------------------------
# host-resident entry points: CPU tensors in/out, PCIe overlapped with the
# kernels (fc2_encode_host / fc2_decode_host / fc2_roundtrip_host)
# ---------------------------------------------------------------------------


def _host_tensor(t, what):
    if not isinstance(t, torch.Tensor) or t.is_cuda or not t.is_contiguous():
        raise TypeError(f"{what} must be a contiguous CPU tensor (pinned for overlap)")
    return t


def encode_host(x: torch.Tensor, config: QuantConfig, payload: torch.Tensor | None = None,
                slice_elems: int = 1 << 22, check: bool = True) -> torch.Tensor:
    """encode_chunk of a host-resident chunk (codec.py:477-519): CPU bf16 /
    float32 / float64 tensor of n elements (n % group_size == 0) -> uint8 CPU
    payload (planes, then metadata).  Stream-ordered; with ``check`` the call
    synchronizes and raises the reference's errors."""
    dev = _device.require_cuda()
    if config.int_log:
        _device.ensure_intlog(config.theta, dev)
    x = _host_tensor(x, "x").reshape(-1)
    n = x.numel()
    F = footprint_bytes(config, n)
    if payload is None:
        payload = torch.empty(F, dtype=torch.uint8, pin_memory=True)
    _host_tensor(payload, "payload")
    xd = _device.workspace("host_x", n * x.element_size(), dev)
    pd = _device.workspace("host_pay", F, dev)
    err = _device.workspace("host_err", 4, dev)[:4].view(torch.int32)
    err.zero_()
    cfg = config.c_struct()
    _lib.check(_lib.lib().fc2_encode_host(ctypes.byref(cfg), x.data_ptr(), _device.dtype_code(x), n,
                                          xd.data_ptr(), pd.data_ptr(), payload.data_ptr(), int(slice_elems),
                                          err.data_ptr(), _device.stream_handle()))
    if check:
        torch.cuda.current_stream().synchronize()
        _device.check_err(err)
    return payload


def decode_host(payload: torch.Tensor, config: QuantConfig, n: int, out: torch.Tensor | None = None,
                out_dtype: torch.dtype = torch.float32, slice_elems: int = 1 << 22,
                check: bool = True) -> torch.Tensor:
    """decode_chunk of a host-resident payload (codec.py:522-563) into a CPU
    tensor of ``out_dtype`` (bf16 / float32 / float64)."""
    dev = _device.require_cuda()
    if config.int_log:
        _device.ensure_intlog(config.theta, dev)
    payload = _host_tensor(payload, "payload")
    F = footprint_bytes(config, n)
    if payload.numel() < F:
        raise DecodeFormatError(f"payload has {payload.numel()} bytes, chunk needs {F}")
    if out is None:
        out = torch.empty(n, dtype=out_dtype, pin_memory=True)
    _host_tensor(out, "out")
    pd = _device.workspace("host_pay", F, dev)
    yd = _device.workspace("host_y", n * out.element_size(), dev)
    err = _device.workspace("host_err", 4, dev)[:4].view(torch.int32)
    err.zero_()
    cfg = config.c_struct()
    _lib.check(_lib.lib().fc2_decode_host(ctypes.byref(cfg), payload.data_ptr(), n, pd.data_ptr(), yd.data_ptr(),
                                          _device.dtype_code(out), out.data_ptr(), int(slice_elems),
                                          err.data_ptr(), _device.stream_handle()))
    if check:
        torch.cuda.current_stream().synchronize()
        _device.check_err(err)
    return out


def roundtrip_host(x: torch.Tensor, config: QuantConfig, payload: torch.Tensor | None = None,
                   out: torch.Tensor | None = None, out_dtype: torch.dtype | None = None,
                   slice_elems: int = 1 << 22, check: bool = True):
    """Encode then decode a host-resident chunk in one pipelined pass (the
    QDQ of collectives.py:179-182): returns (payload, decoded) CPU tensors;
    pass ``payload=False`` to skip copying the packed bytes back."""
    dev = _device.require_cuda()
    if config.int_log:
        _device.ensure_intlog(config.theta, dev)
    x = _host_tensor(x, "x").reshape(-1)
    n = x.numel()
    F = footprint_bytes(config, n)
    if payload is None:
        payload = torch.empty(F, dtype=torch.uint8, pin_memory=True)
    if out is None:
        out = torch.empty(n, dtype=out_dtype or x.dtype, pin_memory=True)
    _host_tensor(out, "out")
    xd = _device.workspace("host_x", n * x.element_size(), dev)
    pd = _device.workspace("host_pay", F, dev)
    yd = _device.workspace("host_y", n * out.element_size(), dev)
    err = _device.workspace("host_err", 4, dev)[:4].view(torch.int32)
    err.zero_()
    cfg = config.c_struct()
    ph = 0 if payload is False else _host_tensor(payload, "payload").data_ptr()
    _lib.check(_lib.lib().fc2_roundtrip_host(ctypes.byref(cfg), x.data_ptr(), _device.dtype_code(x), n,
                                             xd.data_ptr(), pd.data_ptr(), yd.data_ptr(), _device.dtype_code(out),
                                             ph, out.data_ptr(), int(slice_elems), err.data_ptr(),
                                             _device.stream_handle()))
    if check:
        torch.cuda.current_stream().synchronize()
        _device.check_err(err)
    return (None if payload is False else payload), out


# ---------------------------------------------------------------------------
# reference-named API
# ---------------------------------------------------------------------------


def encode_chunk(values, config: QuantConfig) -> QuantizedChunk:
    """Encode ``config.chunk_size`` values into a chunk (codec.py:477-519)."""
    dev = _device.require_cuda()
    device_in = _device.is_cuda_tensor(values)
    if device_in:
        x = values.detach()
        if x.dtype not in (torch.bfloat16, torch.float32, torch.float64):
            x = x.to(torch.float64)
        if x.dim() != 1 or x.numel() != config.chunk_size:
            raise DataError(f"expected {config.chunk_size} values, got shape {tuple(x.shape)}")
        x = x.contiguous()
    else:
        arr = np.asarray(values) if not isinstance(values, torch.Tensor) else values.numpy()
        if arr.ndim != 1 or arr.size != config.chunk_size:
            raise DataError(f"expected {config.chunk_size} values, got shape {arr.shape}")
        x = _device.to_device_values(arr, dev)
    payload = encode_payload(x, config, config.chunk_size)
    if device_in:
        return QuantizedChunk(config, element_count=config.chunk_size, payload=payload)
    chunk = QuantizedChunk(config, element_count=config.chunk_size, payload=payload)
    chunk._materialize()
    chunk._payload = None  # host residency: bytes only, like the reference
    return chunk


def decode_chunk(chunk: QuantizedChunk, out_dtype=None):
    """Invert :func:`encode_chunk` (codec.py:522-563).

    Host chunks decode to float64 numpy (bit-identical to the reference);
    device chunks decode to a CUDA tensor (float32 unless ``out_dtype``)."""
    config = chunk.config
    n = chunk.element_count
    host = not chunk.on_device
    if host:
        units = bit_split(config.bitwidth)
        if len(chunk.planes) != len(units):
            raise DecodeFormatError(f"expected {len(units)} planes, got {len(chunk.planes)}")
        for p, w in zip(chunk.planes, units):
            if len(p) != n * w // 8:
                raise DecodeFormatError(f"plane of width {w} has {len(p)} bytes, expected {n * w // 8}")
        if n % config.group_size:
            raise DecodeFormatError("element count not a multiple of group size")
        expected = (n // config.group_size) * meta_record_nbytes(config)
        if len(chunk.meta) != expected:
            raise DecodeFormatError(f"metadata has {len(chunk.meta)} bytes, expected {expected}")
    dt = out_dtype or (torch.float64 if host else torch.float32)
    y = decode_payload(chunk.payload, config, n, out_dtype=dt)
    if not host:
        return y
    chunk._payload = None  # keep host residency
    return y.cpu().numpy()


def pack_codes(codes, bitwidth: int) -> list[bytes]:
    """Pack integer codes into one byte plane per bit-split unit (codec.py:204-225)."""
    from .errors import CodeRangeError

    units = bit_split(bitwidth)
    arr = np.asarray(codes)
    if arr.ndim != 1:
        raise DataError("codes must be one-dimensional")
    if arr.size % 8 != 0:
        raise DataError(f"code count {arr.size} must be a multiple of 8")
    if arr.size == 0:
        return [b"" for _ in units]
    if arr.dtype.kind not in "iub":
        arr = arr.astype(np.int64)
    big = arr.astype(np.int64)
    dev = _device.require_cuda()
    if np.any(big != arr):
        raise CodeRangeError(f"codes out of range for {bitwidth}-bit encoding")
    d_codes = torch.from_numpy(np.ascontiguousarray(big)).to(dev)
    n = arr.size
    out = torch.empty(n * bitwidth // 8, dtype=torch.uint8, device=dev)
    err = _device.new_err(dev)
    _lib.check(_lib.lib().fc2_pack_codes(d_codes.data_ptr(), n, bitwidth, out.data_ptr(),
                                         err.data_ptr(), _device.stream_handle()))
    _device.check_err(err)
    raw = out.cpu().numpy().tobytes()
    planes, pos = [], 0
    for w in units:
        planes.append(raw[pos:pos + n * w // 8])
        pos += n * w // 8
    return planes


def unpack_codes(planes, bitwidth: int, count: int) -> np.ndarray:
    """Exact inverse of :func:`pack_codes` (codec.py:228-238)."""
    units = bit_split(bitwidth)
    if len(planes) != len(units):
        raise DecodeFormatError(f"expected {len(units)} planes, got {len(planes)}")
    for p, w in zip(planes, units):
        if len(p) != count * w // 8:
            raise DecodeFormatError(
                f"plane of width {w} has {len(p)} bytes, expected {count * w // 8}")
    if count == 0:
        return np.zeros(0, dtype=np.uint8)
    if count % 8:
        raise DecodeFormatError("count must be a multiple of 8")
    dev = _device.require_cuda()
    buf = np.frombuffer(b"".join(bytes(p) for p in planes), dtype=np.uint8)
    d_in = torch.from_numpy(buf.copy()).to(dev)
    d_out = torch.empty(count, dtype=torch.uint8, device=dev)
    _lib.check(_lib.lib().fc2_unpack_codes(d_in.data_ptr(), count, bitwidth, d_out.data_ptr(),
                                           _device.stream_handle()))
    return d_out.cpu().numpy()


# ---------------------------------------------------------------------------
# per-group scalar API (codec.py:278-343) and integer log scales (:366-392)
# ---------------------------------------------------------------------------


def _group_f64(values) -> torch.Tensor:
    v = np.asarray(values.detach().cpu() if isinstance(values, torch.Tensor) else values, dtype=np.float64)
    if v.ndim != 1 or v.size < 1:
        raise DataError("group must be a non-empty one-dimensional vector")
    dev = _device.require_cuda()
    return torch.from_numpy(np.ascontiguousarray(v)).to(dev)


def _levels_check(bitwidth: int) -> None:
    if not 2 <= bitwidth <= 8:
        raise ConfigError(f"bitwidth must be in [2, 8], got {bitwidth}")


def _group_encode(values, bitwidth: int, sr: bool):
    _levels_check(bitwidth)
    x = _group_f64(values)
    n = x.numel()
    if sr and n < 4:
        raise ConfigError(f"spike reserving needs at least 4 elements, got {n}")
    codes = torch.empty(n, dtype=torch.uint8, device=x.device)
    params = torch.zeros(4, dtype=torch.float64, device=x.device)
    idx = torch.zeros(2, dtype=torch.int32, device=x.device)
    err = _device.new_err(x.device)
    _lib.check(_lib.lib().fc2_group_encode_raw(x.data_ptr(), n, bitwidth, int(sr), codes.data_ptr(),
                                               params.data_ptr(), idx.data_ptr(), err.data_ptr(),
                                               _device.stream_handle()))
    _device.check_err(err, "group ")
    return codes.cpu().numpy(), params.cpu().numpy(), idx.cpu().numpy()


def rtn_encode_group(values, bitwidth: int):
    """Asymmetric round-to-nearest over one group -> (codes, scale, zero) (codec.py:278-290)."""
    codes, params, _ = _group_encode(values, bitwidth, sr=False)
    return codes, float(params[0]), float(params[1])


def rtn_decode_group(codes, scale: float, zero: float) -> np.ndarray:
    """codes * scale + zero in float64 (codec.py:293-295)."""
    c = np.ascontiguousarray(np.asarray(codes).astype(np.uint8).reshape(-1))
    if c.size == 0:
        return np.zeros(0)
    dev = _device.require_cuda()
    dc = torch.from_numpy(c).to(dev)
    out = torch.empty(c.size, dtype=torch.float64, device=dev)
    _lib.check(_lib.lib().fc2_group_decode_raw(dc.data_ptr(), c.size, float(scale), float(zero), out.data_ptr(),
                                               _device.stream_handle()))
    return out.cpu().numpy()


def spike_encode_group(values, bitwidth: int):
    """Quantize one group with its first min / max reserved -> (codes, GroupMeta) (codec.py:298-329)."""
    codes, params, idx = _group_encode(values, bitwidth, sr=True)
    meta = GroupMeta(scale=float(params[0]), zero=float(params[1]), spike_min_value=float(params[2]),
                     spike_max_value=float(params[3]), spike_min_index=int(idx[0]), spike_max_index=int(idx[1]))
    return codes, meta


def spike_decode_group(codes, meta: GroupMeta) -> np.ndarray:
    """Dequantize and restore the reserved min / max (codec.py:332-343)."""
    out = rtn_decode_group(codes, meta.scale, meta.zero)
    g = out.size
    if not (0 <= meta.spike_min_index < g and 0 <= meta.spike_max_index < g):
        raise DecodeFormatError(
            f"spike indices ({meta.spike_min_index}, {meta.spike_max_index}) out of range for group of {g}")
    out[meta.spike_min_index] = meta.spike_min_value
    out[meta.spike_max_index] = meta.spike_max_value
    return out


def scale_to_int(scale, theta: int = 10):
    """round-half-away(log2(scale) * theta) clipped to int8; 0 -> -128 (codec.py:366-381)."""
    s = np.asarray(scale, dtype=np.float64)
    dev = _device.require_cuda()
    flat = torch.from_numpy(np.ascontiguousarray(s.reshape(-1))).to(dev)
    out = torch.empty(flat.numel(), dtype=torch.int8, device=dev)
    err = _device.new_err(dev)
    if flat.numel():
        _lib.check(_lib.lib().fc2_scale_to_int(flat.data_ptr(), flat.numel(), int(theta), out.data_ptr(),
                                               err.data_ptr(), _device.stream_handle()))
    _device.check_err(err)
    res = out.cpu().numpy().reshape(s.shape)
    return int(res) if np.ndim(scale) == 0 else res


def int_to_scale(si, theta: int = 10):
    """2 ** (si / theta); the -128 sentinel decodes to 0 (codec.py:384-392)."""
    if theta <= 0:
        raise ConfigError(f"theta must be positive, got {theta}")
    v = np.asarray(si, dtype=np.float64)
    dev = _device.require_cuda()
    _device.ensure_intlog(int(theta), dev)
    flat = torch.from_numpy(np.ascontiguousarray(v.reshape(-1))).to(dev)
    out = torch.empty(flat.numel(), dtype=torch.float64, device=dev)
    if flat.numel():
        _lib.check(_lib.lib().fc2_int_to_scale(flat.data_ptr(), flat.numel(), int(theta), out.data_ptr(),
                                               _device.stream_handle()))
    res = out.cpu().numpy().reshape(v.shape)
    return float(res) if np.ndim(si) == 0 else res
