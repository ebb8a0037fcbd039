"""Tensor and chunk files (reference: fileio.py:1-54), with GPU-batched
quantize / dequantize of whole files.

* ``FCTN`` tensor file: magic, u32 element count, little-endian float32 data
  (fileio.py:17-38).
* Chunk file: serialized ``FCV2`` chunks back to back (fileio.py:41-54); a
  chunk's payload is exactly the device payload (planes, then metadata), so
  serialization is one device->host copy plus a 15-byte header per chunk.

``quantize_tensor`` encodes every chunk of a tensor in batched launches of the
CUDA encoder (one job per chunk, the last chunk may be short, cli.py:79-93);
``dequantize_chunks`` uploads a chunk list once and decodes it in batched
launches (cli.py:104-112).  Results are byte-identical to looping the
reference's ``encode_chunk`` / ``decode_chunk``.
"""

from __future__ import annotations

import struct
from dataclasses import replace
from pathlib import Path

import numpy as np
import torch

from . import _device
from .codec import QuantizedChunk, parse_chunk
from .collectives import _decode_jobs, _encode_jobs
from .config import QuantConfig, bit_split, footprint_bytes
from .errors import DataError, DecodeFormatError

TENSOR_MAGIC = b"FCTN"
_TENSOR_HEADER = struct.Struct("<4sI")

__all__ = ["TENSOR_MAGIC", "write_tensor", "read_tensor", "write_chunks", "read_chunks",
           "quantize_tensor", "dequantize_chunks"]


def write_tensor(path, values) -> None:
    arr = np.asarray(values.cpu() if isinstance(values, torch.Tensor) else values, dtype="<f4").reshape(-1)
    with open(path, "wb") as fh:
        fh.write(_TENSOR_HEADER.pack(TENSOR_MAGIC, arr.size))
        fh.write(arr.tobytes())


def read_tensor(path) -> np.ndarray:
    buf = Path(path).read_bytes()
    if len(buf) < _TENSOR_HEADER.size:
        raise DecodeFormatError(f"{path}: too short for a tensor header")
    magic, count = _TENSOR_HEADER.unpack_from(buf, 0)
    if magic != TENSOR_MAGIC:
        raise DecodeFormatError(f"{path}: bad magic {magic!r}")
    expected = _TENSOR_HEADER.size + 4 * count
    if len(buf) != expected:
        raise DecodeFormatError(f"{path}: expected {expected} bytes, found {len(buf)}")
    return np.frombuffer(buf, dtype="<f4", count=count, offset=_TENSOR_HEADER.size).copy()


def write_chunks(path, chunks) -> None:
    with open(path, "wb") as fh:
        for chunk in chunks:
            fh.write(chunk.to_bytes())


def read_chunks(path) -> list[QuantizedChunk]:
    buf = Path(path).read_bytes()
    chunks, pos = [], 0
    while pos < len(buf):
        chunk, pos = parse_chunk(buf, pos)
        chunks.append(chunk)
    return chunks


def _chunk_bounds(n: int, chunk_size: int):
    pos = 0
    while pos < n:
        size = min(chunk_size, n - pos)
        yield pos, size
        pos += size


def quantize_tensor(values, config: QuantConfig, device_payload: bool = False) -> list[QuantizedChunk]:
    """Encode ``values`` as consecutive chunks of ``config.chunk_size``
    elements (the last one may be shorter), like the reference CLI's
    ``quantize`` loop (cli.py:79-93).  All chunks are encoded on the GPU in
    batched launches; host chunks are returned unless ``device_payload``."""
    dev = _device.require_cuda()
    if config.int_log:
        _device.ensure_intlog(config.theta, dev)
    x = _device.to_device_values(values, dev).reshape(-1)
    n = x.numel()
    if n % config.group_size:
        raise DataError(f"tensor has {n} elements, not a multiple of group size {config.group_size}")
    bounds = list(_chunk_bounds(n, config.chunk_size))
    sizes = [footprint_bytes(config, s) for _, s in bounds]
    # every chunk gets a 16-byte aligned slot (the encoder stores whole words;
    # footprints such as 19 or 1938 bytes are not word multiples); the chunks
    # are sliced back to their exact footprints below
    slots = [(f + 15) // 16 * 16 for f in sizes]
    offs = np.concatenate([[0], np.cumsum(slots)]).astype(np.int64)
    out = torch.empty(max(int(offs[-1]), 1), dtype=torch.uint8, device=dev)
    err = _device.new_err(dev)
    es = x.element_size()
    jobs = [(x.data_ptr() + p * es, s, s, out.data_ptr() + int(offs[i])) for i, (p, s) in enumerate(bounds)]
    _encode_jobs(config, _device.dtype_code(x), jobs, err)
    _device.check_err(err)
    chunks = []
    if device_payload:
        for i, (_, s) in enumerate(bounds):
            chunks.append(QuantizedChunk(replace(config, chunk_size=s), element_count=s,
                                         payload=out[int(offs[i]):int(offs[i]) + sizes[i]]))
        return chunks
    host = out.cpu().numpy()
    for i, (_, s) in enumerate(bounds):
        c = QuantizedChunk(replace(config, chunk_size=s), element_count=s,
                           payload=torch.from_numpy(host[int(offs[i]):int(offs[i]) + sizes[i]]))
        c._materialize()
        c._payload = None
        chunks.append(c)
    return chunks


def dequantize_chunks(chunks, out_dtype=np.float64):
    """Decode a list of chunks into one concatenated array (cli.py:104-112):
    float64 numpy by default (bit-identical to the reference's
    ``np.concatenate([decode_chunk(c) ...])``), or a CUDA tensor when
    ``out_dtype`` is a torch dtype."""
    if not chunks:
        raise DecodeFormatError("no chunks to decode")
    dev = _device.require_cuda()
    device_out = isinstance(out_dtype, torch.dtype)
    tdt = out_dtype if device_out else {np.float64: torch.float64, np.float32: torch.float32}[np.dtype(out_dtype).type]
    counts = [c.element_count for c in chunks]
    pos = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    y = torch.empty(int(pos[-1]), dtype=tdt, device=dev)
    err = _device.new_err(dev)
    host = [c for c in chunks if not c.on_device]
    if host:  # one upload for every host chunk (a chunk's bytes are planes + meta)
        for c in host:
            if len(c.planes) != len(bit_split(c.config.bitwidth)):
                raise DecodeFormatError("chunk plane count does not match its bitwidth")
        # each chunk at a 16-byte aligned slot so the vectorised decoder applies
        parts = []
        for c in host:
            b = b"".join(c.planes) + c.meta
            parts.append(b + bytes(-len(b) % 16))
        blob = np.frombuffer(b"".join(parts), dtype=np.uint8)
        dblob = torch.from_numpy(blob.copy()).to(dev)
    groups: dict = {}
    hoff = 0
    for i, c in enumerate(chunks):
        if c.on_device:
            ptr = c.payload.data_ptr()
        else:
            want = footprint_bytes(c.config, c.element_count)
            if c.payload_nbytes != want:
                raise DecodeFormatError(f"chunk {i} holds {c.payload_nbytes} payload bytes, expected {want}")
            ptr = dblob.data_ptr() + hoff
            hoff += (want + 15) // 16 * 16
        key = replace(c.config, chunk_size=c.config.group_size)
        groups.setdefault(key, []).append((ptr, c.element_count, y.data_ptr() + int(pos[i]) * y.element_size(),
                                           c.element_count))
    for cfg, jobs in groups.items():
        if cfg.int_log:
            _device.ensure_intlog(cfg.theta, dev)
        _decode_jobs(cfg, _device.dtype_code(y), jobs, err)
    _device.check_err(err)
    return y if device_out else y.cpu().numpy()

