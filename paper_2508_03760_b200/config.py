"""Codec configuration and byte accounting (host-side; no compute).

Mirrors codec.py:40-102, 143-162, 400-451 of the reference: same names, same
validation messages/exception types, same footprint arithmetic.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

from . import _lib
from .errors import ConfigError

_BIT_SPLIT = {2: (2,), 3: (2, 1), 4: (4,), 5: (4, 1), 6: (4, 2), 7: (4, 2, 1), 8: (8,)}


class Scheme(Enum):
    RTN = "rtn"
    SPIKE_RESERVING = "sr"


class ScaleEncoding(Enum):
    BF16 = "bf16"
    INT_LOG = "intlog"


def default_group_size(bitwidth: int) -> int:
    """128 at 5+ bits, 32 below (codec.py:50-52)."""
    return 128 if bitwidth >= 5 else 32


@dataclass(frozen=True)
class QuantConfig:
    """Parameters of one codec run (codec.py:55-90)."""

    bitwidth: int
    group_size: int | None = None
    scheme: Scheme = Scheme.RTN
    scale_encoding: ScaleEncoding = ScaleEncoding.BF16
    theta: int = 10
    chunk_size: int = 4096

    def __post_init__(self):
        if not 2 <= self.bitwidth <= 8:
            raise ConfigError(f"bitwidth must be in [2, 8], got {self.bitwidth}")
        if self.group_size is None:
            object.__setattr__(self, "group_size", default_group_size(self.bitwidth))
        gs = self.group_size
        if gs <= 0 or gs % 8 != 0:
            raise ConfigError(f"group_size must be a positive multiple of 8, got {gs}")
        if self.scheme is Scheme.SPIKE_RESERVING and not 4 <= gs <= 256:
            raise ConfigError(f"spike reserving needs 4 <= group_size <= 256, got {gs}")
        if self.chunk_size <= 0 or self.chunk_size % gs != 0:
            raise ConfigError(
                f"chunk_size {self.chunk_size} must be a positive multiple of group_size {gs}"
            )
        if not 1 <= self.theta <= 255:
            raise ConfigError(f"theta must be in [1, 255], got {self.theta}")

    @property
    def levels(self) -> int:
        return (1 << self.bitwidth) - 1

    @property
    def spike_reserving(self) -> bool:
        return self.scheme is Scheme.SPIKE_RESERVING

    @property
    def int_log(self) -> bool:
        return self.scale_encoding is ScaleEncoding.INT_LOG

    def c_struct(self) -> _lib.Config:
        return _lib.Config(self.bitwidth, self.group_size, 1 if self.spike_reserving else 0,
                           1 if self.int_log else 0, self.theta)


@dataclass(frozen=True)
class GroupMeta:
    """Decoded per-group metadata; spike fields are None under RTN (codec.py:93-102)."""

    scale: float
    zero: float
    spike_min_value: float | None = None
    spike_max_value: float | None = None
    spike_min_index: int | None = None
    spike_max_index: int | None = None


def bit_split(bitwidth: int) -> list[int]:
    """Unit widths, low bits first: 5 -> [4, 1], 7 -> [4, 2, 1] (codec.py:154-162)."""
    if bitwidth not in _BIT_SPLIT:
        raise ConfigError(f"bitwidth must be in [2, 8], got {bitwidth}")
    return list(_BIT_SPLIT[bitwidth])


def meta_record_nbytes(config: QuantConfig) -> int:
    """Metadata bytes per group (codec.py:400-425)."""
    if config.int_log:
        return 8 if config.spike_reserving else 2
    return 12 if config.spike_reserving else 4


def footprint_bytes(config: QuantConfig, n: int) -> int:
    """Exact payload size (codes + metadata) for n elements (codec.py:428-432)."""
    if n < 0 or n % config.group_size != 0:
        raise ConfigError(f"element count {n} not a multiple of group_size {config.group_size}")
    return n * config.bitwidth // 8 + (n // config.group_size) * meta_record_nbytes(config)


def footprint_breakdown(config: QuantConfig, n: int) -> dict:
    """Codes / scale-zero / spikes / totals (codec.py:435-451)."""
    if n < 0 or n % config.group_size != 0:
        raise ConfigError(f"element count {n} not a multiple of group_size {config.group_size}")
    groups = n // config.group_size
    scale_zero = groups * (2 if config.int_log else 4)
    spikes = groups * (6 if config.int_log else 8) if config.spike_reserving else 0
    quantized = n * config.bitwidth // 8
    return {
        "quantized": quantized,
        "scale_zero": scale_zero,
        "spikes": spikes,
        "meta": scale_zero + spikes,
        "total": quantized + scale_zero + spikes,
    }


def plane_sizes(config: QuantConfig, n: int) -> list[int]:
    """Byte length of each bit-split plane for n elements."""
    return [n * w // 8 for w in bit_split(config.bitwidth)]
