"""Pin the CPU oracle (oracle/fc2_oracle.py) against the reference.

Two sources: (1) golden fixtures produced by running the real reference
(tests/golden/make_golden.py), compared byte-for-byte; (2) the reference's own
known-answer tests, restated here with their file:line.
"""

import hashlib
import struct

import numpy as np
import pytest

from oracle import fc2_oracle as O
from tests.golden_io import load


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


CODEC, CODEC_IDX = load("codec_golden.npz")


@pytest.mark.parametrize("case", CODEC_IDX, ids=[c["key"] for c in CODEC_IDX])
def test_oracle_codec_bytes_match_reference(case):
    x = CODEC[case["input"]]
    planes, meta = O.encode(x, case["bits"], case["g"], case["sr"], case["intlog"])
    got = np.frombuffer(b"".join(planes) + meta, dtype=np.uint8)
    want = CODEC["payload_" + case["key"]]
    assert [len(p) for p in planes] == case["planes"] and len(meta) == case["meta"]
    assert np.array_equal(got, want)
    dec = O.decode(planes, meta, x.size, case["bits"], case["g"], case["sr"], case["intlog"])
    assert sha(dec) == case["decoded_sha"]


TS, TS_IDX = load("two_step_golden.npz")


@pytest.mark.parametrize("case", [c for c in TS_IDX if c["key"] != "ts_identical"],
                         ids=lambda c: c["key"])
def test_oracle_two_step_matches_reference(case):
    payloads = list(TS["in_" + case["key"]])
    outs, nbytes = O.two_step(payloads, case["bits"], case["g"], case["sr"])
    assert np.array_equal(outs[0], TS["out_" + case["key"]])
    N = case["N"]
    # actual bytes == 2 N (N-1) F(shard)  (test_collectives.py:82-88)
    assert case["total_actual"] == 2 * N * (N - 1) * nbytes


def test_oracle_two_step_identical_payloads():
    p = TS["in_ts_identical"]
    outs, _ = O.two_step([p.copy() for _ in range(8)], 5, 128, False)
    assert np.array_equal(outs[0], TS["out_ts_identical"])


A2A, A2A_IDX = load("a2a_golden.npz")


@pytest.mark.parametrize("case", A2A_IDX, ids=lambda c: c["key"])
def test_oracle_a2a_matches_reference(case):
    key, N = case["key"], case["N"]
    payloads = [A2A[f"in_{key}_{i}"] for i in range(N)]
    mat = A2A[f"matrix_{key}"] if case["matrix"] else None
    out = O.a2a_dispatch(payloads, case["bits"], case["g"], case["sr"], mat)
    flat = np.concatenate([out[d][s] for d in range(N) for s in range(N)])
    assert np.array_equal(flat, A2A["out_" + key])


# --- the reference's own known-answer tests, restated -----------------------


def test_kat_five_bit_plane():
    # test_bit_packing.py:26-31
    planes = O.pack([31, 0, 16, 1, 15, 2, 8, 4], 5)
    assert planes[0] == bytes([0x0F, 0x10, 0x2F, 0x48])
    assert list(O.unpack(planes, 5, 8)) == [31, 0, 16, 1, 15, 2, 8, 4]


def test_kat_constant_sr_chunk_bytes():
    # test_chunk_codec.py:112-122 (payload part; the 15-byte header is host-only)
    planes, meta = O.encode(np.full(32, 5.0), 2, 32, sr=True)
    assert planes == [bytes(8)]
    assert meta == struct.pack("<HHHHHH", 0x0000, 0x40A0, 0x40A0, 0x40A0, 0x0000, 0x3F80)
    assert list(O.decode(planes, meta, 32, 2, 32, sr=True)) == [5.0] * 32


@pytest.mark.parametrize("sr,intlog,total", [(True, False, 2560), (True, True, 2048)])
def test_kat_table5_footprints(sr, intlog, total):
    # test_chunk_codec.py:54-64
    assert O.footprint(2, 32, sr, intlog, 4096) == total


def test_kat_int8_rtn_footprint():
    assert O.footprint(8, 128, False, False, 4096) == 4224  # test_chunk_codec.py:67-68


def test_kat_rtn_ties_away_from_zero():
    # test_rtn_groups.py:65-70: [0, .5, 2.5, 3] @2 bits -> [0, 1, 3, 3]
    planes, meta = O.encode([0.0, 0.5, 2.5, 3.0] * 2, 2, 8)
    assert list(O.unpack(planes, 2, 8)[:4]) == [0, 1, 3, 3]


def test_kat_rtn_endpoints():
    # test_rtn_groups.py:27-31: [-2, 2] @8 bits -> codes 0 / 255
    planes, _ = O.encode([-2.0, 2.0] * 4, 8, 8)
    assert list(O.unpack(planes, 8, 8)[:2]) == [0, 255]


def test_kat_bf16_patterns():
    # test_bfloat16.py:11-32
    assert int(O.bf16_bits(np.float32(1.0))) == 0x3F80
    assert int(O.bf16_bits(np.float32(5.0))) == 0x40A0
    assert int(O.bf16_bits(np.float32(-2.0))) == 0xC000
    half = np.frombuffer((0x3F808000).to_bytes(4, "little"), "<f4")[0]
    assert int(O.bf16_bits(half)) == 0x3F80
    half2 = np.frombuffer((0x3F818000).to_bytes(4, "little"), "<f4")[0]
    assert int(O.bf16_bits(half2)) == 0x3F82
    assert O.bf16_snap(np.finfo(np.float32).max) == np.inf


@pytest.mark.parametrize("bits", range(2, 9))
def test_pack_matches_bitwise_definition(bits):
    # test_bit_packing.py:68-72 (bit-by-bit oracle, restated)
    rng = np.random.default_rng(bits)
    codes = rng.integers(0, 1 << bits, 64)
    planes, off = [], 0
    for w in O.UNITS[bits]:
        bitstream = [(int(c) >> (off + b)) & 1 for c in codes for b in range(w)]
        plane = bytearray(len(bitstream) // 8)
        for i, bit in enumerate(bitstream):
            plane[i // 8] |= bit << (i % 8)
        planes.append(bytes(plane))
        off += w
    assert O.pack(codes, bits) == planes


def test_synthetic_stream_pinned():
    # test_synthetic.py:15-21: n=4096, seed 2024, rate 1/32 lands on 133 spikes
    v = O.spiky(4096, 2024, rate=1 / 32)
    assert int(np.sum(np.abs(v) >= 49.0)) == 133


GRP, GRP_IDX = load("group_golden.npz")


def test_oracle_group_api_matches_reference():
    # codec.py:278-343 per-group API vs the reference's own outputs
    for c in GRP_IDX:
        g = GRP[f"g{c['i']}"]
        codes, s, z = O.rtn_group(g, c["bits"])
        assert np.array_equal(codes, GRP[f"rtn{c['i']}_b{c['bits']}"])
        assert (s, z) == (c["rtn_scale"], c["rtn_zero"])
        codes, s, z, a, b, ia, ib = O.spike_group(g, c["bits"])
        assert np.array_equal(codes, GRP[f"sr{c['i']}_b{c['bits']}"])
        assert (s, z, a, b, ia, ib) == (c["sr_scale"], c["sr_zero"], c["smin"], c["smax"], c["imin"], c["imax"])


@pytest.mark.parametrize("theta", [1, 10, 37])
def test_oracle_intlog_helpers_match_reference(theta):
    assert np.array_equal(O.scale_to_int(GRP["scales"], theta), GRP[f"s2i_t{theta}"])
    assert np.array_equal(O.int_to_scale(np.arange(-128, 128), theta), GRP[f"i2s_t{theta}"])
    # known points (test_intlog_scale.py:15-20)
    assert int(O.scale_to_int(1.0)) == 0 and int(O.scale_to_int(2.0)) == 10 and int(O.scale_to_int(0.3)) == -17


HIER, HIER_IDX = load("hier_golden.npz")


@pytest.mark.parametrize("case", HIER_IDX, ids=lambda c: c["key"])
def test_oracle_hierarchical_matches_reference(case):
    """oracle.hierarchical == the reference's hierarchical_two_step_q
    (collectives.py:318-425) on the L40 preset and a 4-GPU bridged fabric."""
    payloads = list(HIER["in_" + case["key"]])
    N = case["N"]
    half = N // 2
    groups = [list(range(half)), list(range(half, N))]
    outs = O.hierarchical(payloads, groups, case["bits"], case["g"], case["sr"])
    want = HIER["out_" + case["key"]]
    for r in range(N):
        assert np.array_equal(outs[r], want[r])
