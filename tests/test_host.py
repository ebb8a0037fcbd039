"""CPU-only tests: host logic of the drop-in API and the C ABI surface.

No compute call happens here (there is no GPU in the build container); the
library is loaded and its exported symbols checked against include/fc2.h.
"""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2508_03760_b200 as fc
from paper_2508_03760_b200 import _lib
from paper_2508_03760_b200.collectives import _two_step_ledger
from tests.golden_io import load

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "fc2.h")).read()
    return sorted(set(re.findall(r"\b(fc2_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    # the ctypes signature table binds exactly the header surface
    assert sorted(_lib.SIGNATURES) == syms
    assert lib.fc2_version() == 1


def test_library_host_entry_points_without_gpu():
    lib = _lib.load()
    c = fc.QuantConfig(4, 128, fc.Scheme.SPIKE_RESERVING).c_struct()
    out = ctypes.c_int64()
    assert lib.fc2_footprint(ctypes.byref(c), 33554432, ctypes.byref(out)) == 0
    assert out.value == 19922944
    assert lib.fc2_meta_offset(ctypes.byref(c), 4096) == 2048
    bad = _lib.Config(9, 128, 0, 0, 10)
    assert lib.fc2_check_config(ctypes.byref(bad)) == _lib.FC2_ECONFIG
    assert b"bitwidth" in lib.fc2_last_error()
    with pytest.raises(fc.ConfigError):
        _lib.check(lib.fc2_check_config(ctypes.byref(bad)))


def test_config_validation_mirrors_reference():
    # codec.py:71-86 / test_chunk_codec.py:43-51
    assert [fc.default_group_size(b) for b in range(2, 9)] == [32, 32, 32, 128, 128, 128, 128]
    for bad in (dict(bitwidth=1), dict(bitwidth=4, group_size=30),
                dict(bitwidth=4, group_size=64, chunk_size=100),
                dict(bitwidth=2, group_size=512, scheme=fc.Scheme.SPIKE_RESERVING, chunk_size=512),
                dict(bitwidth=4, theta=0)):
        with pytest.raises(fc.ConfigError):
            fc.QuantConfig(**bad)
    assert fc.bit_split(7) == [4, 2, 1] and fc.bit_split(3) == [2, 1]
    with pytest.raises(fc.ConfigError):
        fc.bit_split(9)


@pytest.mark.parametrize("sr,enc,expected", [
    (fc.Scheme.SPIKE_RESERVING, fc.ScaleEncoding.BF16, (1024, 512, 1024, 1536, 2560)),
    (fc.Scheme.SPIKE_RESERVING, fc.ScaleEncoding.INT_LOG, (1024, 256, 768, 1024, 2048)),
])
def test_footprint_table5(sr, enc, expected):
    got = fc.footprint_breakdown(fc.QuantConfig(2, group_size=32, scheme=sr, scale_encoding=enc), 4096)
    assert (got["quantized"], got["scale_zero"], got["spikes"], got["meta"], got["total"]) == expected


def test_footprint_baseline_table():
    # 64 MiB bf16, g128
    n = 33554432
    rtn = {2: 9437184, 3: 13631488, 4: 17825792, 5: 22020096, 6: 26214400, 8: 34603008}
    sr = {2: 11534336, 3: 15728640, 4: 19922944, 5: 24117248, 6: 28311552, 8: 36700160}
    for b in rtn:
        assert fc.footprint_bytes(fc.QuantConfig(b, 128), n) == rtn[b]
        assert fc.footprint_bytes(fc.QuantConfig(b, 128, fc.Scheme.SPIKE_RESERVING), n) == sr[b]


def test_chunk_wire_format_roundtrip_host():
    cfg = fc.QuantConfig(2, group_size=32, scheme=fc.Scheme.SPIKE_RESERVING, chunk_size=32)
    import struct
    planes = [bytes(8)]
    meta = struct.pack("<HHHHHH", 0x0000, 0x40A0, 0x40A0, 0x40A0, 0x0000, 0x3F80)
    ch = fc.QuantizedChunk(cfg, planes, meta, 32)
    blob = ch.to_bytes()
    assert blob[:15] == struct.pack("<4sBBHBBBI", b"FCV2", 2, 2, 32, 1, 0, 10, 32)
    assert fc.QuantizedChunk.from_bytes(blob) == ch
    with pytest.raises(fc.DecodeFormatError):
        fc.QuantizedChunk.from_bytes(b"XXXX" + blob[4:])
    with pytest.raises(fc.DecodeFormatError):
        fc.QuantizedChunk.from_bytes(blob[:-1])
    with pytest.raises(fc.DecodeFormatError):
        fc.QuantizedChunk.from_bytes(blob + b"\x00")


TS, TS_IDX = load("two_step_golden.npz")


@pytest.mark.parametrize("case", [c for c in TS_IDX if c["key"] != "ts_identical"], ids=lambda c: c["key"])
def test_two_step_ledger_matches_reference_volumes(case):
    N, n, g = case["N"], case["n"], case["g"]
    cfg = fc.QuantConfig(case["bits"], group_size=g,
                         scheme=fc.Scheme.SPIKE_RESERVING if case["sr"] else fc.Scheme.RTN)
    mult = N * g
    S = -(-n // mult) * mult // N
    topo = fc.preset("H800", N)
    ledger, trace = _two_step_ledger(topo, N, S, fc.footprint_bytes(cfg, S))
    rep = fc.volume_report(ledger, topo)
    assert rep["total_raw"] == case["total_raw"]
    assert rep["total_actual"] == case["total_actual"]
    assert len(ledger.events) == case["events"]


def test_l40_cross_numa_volumes():
    # test_collectives.py:57-61: two-step moves 4M across the NUMA bridge
    topo = fc.preset("L40")
    M = 16384
    cfg = fc.QuantConfig(8)
    S = M // 8
    ledger, _ = _two_step_ledger(topo, 8, S, fc.footprint_bytes(cfg, S))
    rep = fc.volume_report(ledger, topo)
    assert rep["total_raw"] == 14 * 2 * M
    assert rep["cross_numa_raw"] == 4 * 2 * M


def test_hierarchical_is_not_applicable_on_nvswitch():
    with pytest.raises(fc.NotApplicableError):
        fc.hierarchical_two_step_q([np.zeros(8)] * 8, fc.preset("B200"), fc.QuantConfig(8))


def test_topology_json_roundtrip(tmp_path):
    t = fc.preset("L40")
    p = tmp_path / "t.json"
    t.save(p)
    assert fc.Topology.load(p) == t
    with pytest.raises(fc.ConfigError):
        fc.preset("nope")


def test_tie_ge_saturating_form_matches_compare():
    """fc2_common.cuh tie_ge: sat(h - 64992) in f16 (HFMA2.SAT) equals the
    ordered compare h >= 65024 (0x7BF0) for every 16-bit pattern, NaN
    flushing to 0 as .sat does."""
    h = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16).view(np.float16)
    c = float(np.array([0xFBEF], dtype=np.uint16).view(np.float16)[0])
    t = float(np.array([0x7BF0], dtype=np.uint16).view(np.float16)[0])
    assert (c, t) == (-64992.0, 65024.0)
    with np.errstate(all="ignore"):
        r = (h.astype(np.float64) + c).astype(np.float16).astype(np.float64)  # one rounding, as the fma
        sat = np.where(np.isnan(r), 0.0, np.clip(r, 0.0, 1.0))
        ge = (h.astype(np.float64) >= t).astype(np.float64)
    assert np.array_equal(sat, ge)
