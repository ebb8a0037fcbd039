"""GPU parity of the codec (encode_chunk / decode_chunk / pack / unpack).

Bar: bit-exact packed planes, metadata (spike positions and values included)
and decoded values against (1) the reference's own bytes in
tests/golden/codec_golden.npz and (2) the pinned CPU oracle on seeded inputs,
plus size-independent properties at the BASELINE size (64 MiB bf16).
"""

import hashlib

import numpy as np
import pytest
import torch

import paper_2508_03760_b200 as fc
from oracle import fc2_oracle as O
from tests.golden_io import load

pytestmark = pytest.mark.gpu

SCH = {True: fc.Scheme.SPIKE_RESERVING, False: fc.Scheme.RTN}
ENC = {True: fc.ScaleEncoding.INT_LOG, False: fc.ScaleEncoding.BF16}


def cfg_of(bits, g, sr, intlog=False, n=4096):
    return fc.QuantConfig(bits, group_size=g, scheme=SCH[sr], scale_encoding=ENC[intlog], chunk_size=n)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def payload_of(chunk):
    return np.frombuffer(b"".join(chunk.planes) + chunk.meta, dtype=np.uint8)


CODEC, CODEC_IDX = load("codec_golden.npz")


@pytest.mark.parametrize("case", CODEC_IDX, ids=[c["key"] for c in CODEC_IDX])
def test_codec_matches_reference_bytes(case):
    x = CODEC[case["input"]]
    cfg = cfg_of(case["bits"], case["g"], case["sr"], case["intlog"], x.size)
    chunk = fc.encode_chunk(x, cfg)
    assert [len(p) for p in chunk.planes] == case["planes"]
    assert np.array_equal(payload_of(chunk), CODEC["payload_" + case["key"]])
    dec = fc.decode_chunk(chunk)
    assert dec.dtype == np.float64 and sha(dec) == case["decoded_sha"]


@pytest.mark.parametrize("case", [c for c in CODEC_IDX if c["input"] != "in_normal_f64"],
                         ids=lambda c: c["key"])
def test_codec_device_bf16_path_matches_reference(case):
    # bf16-valued inputs encoded from a CUDA bf16 tensor: same bytes
    x = CODEC[case["input"]]
    cfg = cfg_of(case["bits"], case["g"], case["sr"], case["intlog"], x.size)
    xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
    chunk = fc.encode_chunk(xd, cfg)
    assert chunk.on_device
    assert np.array_equal(chunk.payload.cpu().numpy(), CODEC["payload_" + case["key"]])
    dec32 = fc.decode_chunk(chunk)  # float32 on device
    assert sha(dec32.cpu().numpy()) == case["decoded_f32_sha"]


def tie_heavy(n, seed):
    """Values on a coarse grid so (v - zero)/scale hits exact .5 ties often."""
    rng = np.random.default_rng(seed)
    return (rng.integers(-64, 64, n) / 8.0).astype(np.float32)


def stress(n, seed, g=32):
    """Every group of g (the smallest group size of a test: coarser groups mix
    regimes) drawn from a different regime that exercises a separate branch
    of the fast kernels: large offsets (explicit v - off form), tiny and huge
    ranges (the all-float64 path), constant groups (scale 0), many copies of
    both extremes (spike occurrence counting), one-signed groups (the
    reserved-slot stand-in), subnormals, exact-integer grids (near ties)."""
    rng = np.random.default_rng(seed)
    out = np.empty(n, dtype=np.float64)
    regimes = [
        lambda k: rng.normal(0, 1, k),
        lambda k: 1000.0 + rng.normal(0, 1, k),
        lambda k: rng.normal(0, 1e-33, k),
        lambda k: rng.normal(0, 1e30, k),
        lambda k: np.full(k, rng.normal()),
        lambda k: rng.choice([-3.0, 3.0, 0.5], size=k, p=[0.3, 0.3, 0.4]),
        lambda k: np.abs(rng.normal(5, 1, k)) + 1.0,
        lambda k: -np.abs(rng.normal(5, 1, k)) - 1.0,
        lambda k: rng.normal(0, 1e-39, k),
        lambda k: rng.integers(-40, 40, k) / 4.0,
    ]
    for i in range(0, n, g):
        out[i:i + g] = regimes[rng.integers(len(regimes))](min(g, n - i))
    return O.bf16_snap(out.astype(np.float32)).astype(np.float32)


INPUTS = {
    "spiky": lambda n, s: O.bf16_snap(O.spiky(n, s)).astype(np.float32),
    "ties": tie_heavy,
    "gauss_f32": lambda n, s: np.random.default_rng(s).normal(0, 1, n).astype(np.float32),
    "stress": stress,
}


@pytest.mark.parametrize("bits", range(2, 9))
@pytest.mark.parametrize("sr", [False, True])
@pytest.mark.parametrize("g", [32, 64, 128, 256, 24, 40])
@pytest.mark.parametrize("kind", list(INPUTS))
def test_codec_matches_oracle_random(bits, sr, g, kind):
    n = g * 2048
    x = INPUTS[kind](n, bits * 1000 + g)
    cfg = cfg_of(bits, g, sr, False, n)
    chunk = fc.encode_chunk(x, cfg)
    planes, meta = O.encode(x, bits, g, sr)
    assert chunk.planes == planes
    assert chunk.meta == meta
    assert np.array_equal(fc.decode_chunk(chunk), O.decode(planes, meta, n, bits, g, sr))


@pytest.mark.parametrize("bits", range(2, 9))
@pytest.mark.parametrize("sr", [False, True])
@pytest.mark.parametrize("g", [32, 64, 128, 256])
@pytest.mark.parametrize("kind", ["spiky", "ties", "stress"])
def test_codec_bf16_device_matches_oracle(bits, sr, g, kind):
    """The bf16 lane-per-group encoder (k_encode_grp) in its small-chunk
    shape (one 32-element run per lane) against the oracle, every g."""
    n = g * 1024
    x = O.bf16_snap(INPUTS[kind](n, bits * 7 + g)).astype(np.float32)
    cfg = cfg_of(bits, g, sr, False, n)
    chunk = fc.encode_chunk(torch.from_numpy(x).cuda().to(torch.bfloat16), cfg)
    planes, meta = O.encode(x, bits, g, sr)
    assert bytes(chunk.payload.cpu().numpy()) == b"".join(planes) + meta
    dec = fc.decode_payload(chunk.payload, cfg, n, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(dec, O.decode(planes, meta, n, bits, g, sr).astype(np.float32))


@pytest.mark.parametrize("bits", [2, 3, 4, 5, 7, 8])
@pytest.mark.parametrize("sr", [False, True])
@pytest.mark.parametrize("g", [32, 64, 128, 256])
@pytest.mark.parametrize("extra", [0, 3])
def test_codec_bf16_bandwidth_shape_slices(bits, sr, g, extra):
    """The same encoder in its bandwidth shape (chunks of >= one resident
    wave of tiles): slices of the payload equal the oracle on the same
    element slices (groups are independent); extra > 0 leaves a partial last
    warp tile."""
    if extra and bits not in (3, 4):
        pytest.skip("partial last tile: two bit widths are enough")
    n = (1 << 23) + extra * g
    x = torch.from_numpy(O.bf16_snap(O.spiky(n, bits + g)).astype(np.float32)).to(torch.bfloat16)
    cfg = cfg_of(bits, g, sr, False, n)
    ph = fc.encode_payload(x.cuda(), cfg, n).cpu().numpy()
    xs = x.float().numpy()
    rec = 12 if sr else 4
    for start in (0, 3 * 1024 * 1024 + 8192, n - 16384 - extra * g):
        m = 16384 + (extra * g if start > 3 * 1024 * 1024 + 8192 else 0)
        planes, meta = O.encode(xs[start:start + m], bits, g, sr)
        off = 0
        for w, p in zip(O.UNITS[bits], planes):
            assert ph[off + start * w // 8: off + (start + m) * w // 8].tobytes() == p
            off += n * w // 8
        assert ph[off + (start // g) * rec: off + ((start + m) // g) * rec].tobytes() == meta


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
@pytest.mark.parametrize("sr", [False, True])
def test_codec_intlog_matches_oracle(bits, sr):
    n = 128 * 512
    rng = np.random.default_rng(bits)
    x = rng.normal(0, 1, n) * rng.uniform(0.01, 100, n)
    cfg = cfg_of(bits, 128, sr, True, n)
    chunk = fc.encode_chunk(x, cfg)
    planes, meta = O.encode(x, bits, 128, sr, intlog=True)
    assert chunk.planes == planes and chunk.meta == meta
    assert np.array_equal(fc.decode_chunk(chunk), O.decode(planes, meta, n, bits, 128, sr, intlog=True))


@pytest.mark.parametrize("bits,sr,g", [(4, True, 128), (3, True, 128), (8, True, 128), (2, False, 128),
                                        (5, True, 64), (4, True, 256), (6, False, 32)])
def test_codec_bf16_bandwidth_shape_stress(bits, sr, g):
    """The bandwidth shape of k_encode_grp (and k_decode_fast) on the stress
    mix, whole payload and decoded values against the oracle."""
    n = 1 << 22  # above the small-chunk crossover: bandwidth tiles
    x = stress(n, 97 + bits + g, g)
    cfg = cfg_of(bits, g, sr, False, n)
    xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
    pay = fc.encode_payload(xd, cfg, n)
    planes, meta = O.encode(x, bits, g, sr)
    assert np.array_equal(pay.cpu().numpy(), np.frombuffer(b"".join(planes) + meta, dtype=np.uint8))
    dec = fc.decode_payload(pay, cfg, n, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(dec, O.decode(planes, meta, n, bits, g, sr).astype(np.float32))


def test_codec_f64_inputs_are_exact():
    # arbitrary float64 values (not on the f32 grid) use the reference's f64 semantics
    n = 128 * 256
    x = np.random.default_rng(5).normal(0, 1, n) * 1e-3 + 1.0
    for sr in (False, True):
        cfg = cfg_of(4, 128, sr, False, n)
        chunk = fc.encode_chunk(x, cfg)
        planes, meta = O.encode(x, 4, 128, sr)
        assert chunk.planes == planes and chunk.meta == meta


def test_codec_padding_and_partial_tiles():
    # n_valid < n (zero padding) and chunks that are not a multiple of 1024
    for n_valid, n in [(1000, 1024), (5000, 5120), (33, 128), (0, 256), (128 * 9, 128 * 9)]:
        x = O.bf16_snap(O.spiky(max(n_valid, 1), n))[:n_valid].astype(np.float32)
        cfg = cfg_of(4, 128, True, False, n)
        xd = torch.from_numpy(x).cuda()
        pay = fc.encode_payload(xd, cfg, n)
        ref = np.pad(x, (0, n - n_valid))
        planes, meta = O.encode(ref, 4, 128, True)
        assert bytes(pay.cpu().numpy()) == b"".join(planes) + meta


def test_codec_misaligned_device_input():
    # a view starting at an odd element offset takes the generic path
    base = torch.from_numpy(O.bf16_snap(O.spiky(4096 + 3, 9)).astype(np.float32)).cuda()
    x = base[3:]
    cfg = cfg_of(5, 128, True, False, 4096)
    chunk = fc.encode_chunk(x, cfg)
    planes, meta = O.encode(x.cpu().numpy(), 5, 128, True)
    assert chunk.planes == planes and chunk.meta == meta


def test_nonfinite_raises_data_error():
    x = np.arange(256, dtype=np.float32)
    x[77] = np.nan
    for sr in (False, True):
        with pytest.raises(fc.DataError):
            fc.encode_chunk(x, cfg_of(4, 32, sr, False, 256))
    x[77] = np.inf
    with pytest.raises(fc.DataError):
        fc.encode_chunk(torch.from_numpy(x).cuda().to(torch.bfloat16), cfg_of(4, 128, True, False, 256))


def test_bad_spike_index_raises():
    cfg = cfg_of(2, 32, True, False, 32)
    chunk = fc.encode_chunk(np.arange(32, dtype=np.float32), cfg)
    meta = bytearray(chunk.meta)
    meta[10:12] = (0x4300).to_bytes(2, "little")  # bf16 128.0 >= group size
    bad = fc.QuantizedChunk(cfg, chunk.planes, bytes(meta), 32)
    with pytest.raises(fc.DecodeFormatError):
        fc.decode_chunk(bad)


def test_pack_unpack_roundtrip_and_goldens():
    assert fc.pack_codes([31, 0, 16, 1, 15, 2, 8, 4], 5)[0] == bytes([0x0F, 0x10, 0x2F, 0x48])
    rng = np.random.default_rng(3)
    for bits in range(2, 9):
        codes = rng.integers(0, 1 << bits, 8 * 1000)
        planes = fc.pack_codes(codes, bits)
        assert planes == O.pack(codes, bits)
        assert np.array_equal(fc.unpack_codes(planes, bits, codes.size), codes.astype(np.uint8))
    with pytest.raises(fc.CodeRangeError):
        fc.pack_codes([4, 0, 0, 0, 0, 0, 0, 0], 2)
    with pytest.raises(fc.CodeRangeError):
        fc.pack_codes([-1, 0, 0, 0, 0, 0, 0, 0], 3)
    with pytest.raises(fc.DecodeFormatError):
        fc.unpack_codes([b"\x00"], 5, 16)


def test_bf16_helpers_match_reference_patterns():
    assert int(fc.f32_to_bf16_bits(np.float32(1.0))) == 0x3F80
    assert int(fc.f32_to_bf16_bits(np.float32(-2.0))) == 0xC000
    bits = np.arange(0, 1 << 16, dtype=np.uint16)
    f = fc.bf16_bits_to_f32(bits)
    fin = np.isfinite(f)
    assert np.array_equal(fc.f32_to_bf16_bits(f[fin]), bits[fin])
    x = np.random.default_rng(0).normal(0, 1e3, 100000).astype(np.float32)
    assert np.array_equal(fc.bf16_round(x), O.bf16_snap(x))


@pytest.mark.parametrize("bits,sr", [(4, True), (2, True), (3, False), (8, True)])
def test_full_size_64MiB_properties(bits, sr):
    """BASELINE config 2 size (33,554,432 bf16): sampled tiles equal the oracle
    on the same slice (groups are independent), spikes come back exactly and
    every non-spike element is within half a step (+ bf16 metadata slack)."""
    n = 1 << 25
    g = 128
    gen = torch.Generator(device="cuda").manual_seed(bits)
    x = torch.randn(n, device="cuda", generator=gen)
    spike = torch.rand(n, device="cuda", generator=gen) < 1 / 64
    x = torch.where(spike, torch.sign(x) * 50, x).to(torch.bfloat16)
    cfg = cfg_of(bits, g, sr, False, n)
    pay = fc.encode_payload(x, cfg, n)
    y = fc.decode_payload(pay, cfg, n, out_dtype=torch.float32)
    # slices of the payload == oracle on the same element slice
    xs = x.float().cpu().numpy()
    ph = pay.cpu().numpy()
    rec = 12 if sr else 4
    units = O.UNITS[bits]
    for start in (0, 5 * 1024 * 1024 + 4096, n - 8192):
        m = 8192
        planes, meta = O.encode(xs[start:start + m], bits, g, sr)
        off = 0
        for w, p in zip(units, planes):
            got = ph[off + start * w // 8: off + (start + m) * w // 8].tobytes()
            assert got == p
            off += n * w // 8
        gm = ph[off + (start // g) * rec: off + ((start + m) // g) * rec].tobytes()
        assert gm == meta
    # decode == oracle decode of the same slice
    yh = y.cpu().numpy()
    planes, meta = O.encode(xs[:65536], bits, g, sr)
    assert np.array_equal(yh[:65536], O.decode(planes, meta, 65536, bits, g, sr).astype(np.float32))
    # error bound: non-spikes within scale/2 + bf16 slack of the metadata
    err = np.abs(yh - xs).reshape(-1, g)
    rows = xs.reshape(-1, g)
    srt = np.sort(rows, axis=1)
    lo, hi = (srt[:, 1], srt[:, -2]) if sr else (srt[:, 0], srt[:, -1])
    scale = (hi.astype(np.float64) - lo) / ((1 << bits) - 1)
    slack = scale / 2 + ((1 << bits) - 1) * scale * 2.0 ** -8 + np.abs(lo) * 2.0 ** -8 + 1e-30
    body = err.copy()
    if sr:
        body[np.arange(rows.shape[0]), np.argmin(rows, axis=1)] = 0
        body[np.arange(rows.shape[0]), np.argmax(rows, axis=1)] = 0
    assert np.all(body.max(axis=1) <= slack * (1 + 1e-6))


GRP, GRP_IDX = load("group_golden.npz")


def test_group_api_matches_reference():
    # rtn_/spike_encode_group and decoders (codec.py:278-343) on the GPU
    for c in GRP_IDX:
        g = GRP[f"g{c['i']}"]
        codes, s, z = fc.rtn_encode_group(g, c["bits"])
        assert np.array_equal(codes, GRP[f"rtn{c['i']}_b{c['bits']}"])
        assert (s, z) == (c["rtn_scale"], c["rtn_zero"])
        assert np.array_equal(fc.rtn_decode_group(codes, s, z), O.group_decode(codes, s, z))
        codes, m = fc.spike_encode_group(g, c["bits"])
        assert np.array_equal(codes, GRP[f"sr{c['i']}_b{c['bits']}"])
        assert (m.scale, m.zero, m.spike_min_value, m.spike_max_value, m.spike_min_index, m.spike_max_index) == \
            (c["sr_scale"], c["sr_zero"], c["smin"], c["smax"], c["imin"], c["imax"])
        want = O.group_decode(codes, m.scale, m.zero)
        want[m.spike_min_index] = m.spike_min_value
        want[m.spike_max_index] = m.spike_max_value
        assert np.array_equal(fc.spike_decode_group(codes, m), want)
    with pytest.raises(fc.ConfigError):
        fc.spike_encode_group([1.0, 2.0, 3.0], 2)
    with pytest.raises(fc.DataError):
        fc.rtn_encode_group([1.0, float("nan")], 4)
    with pytest.raises(fc.DecodeFormatError):
        fc.spike_decode_group(np.zeros(8, np.uint8), fc.GroupMeta(1.0, 0.0, 0.0, 1.0, 0, 99))


@pytest.mark.parametrize("theta", [1, 10, 37])
def test_intlog_helpers_match_reference(theta):
    # bit-exact except where log2(scale)*theta is within 1e-9 of a .5 rounding
    # tie: there the result depends on the last ulp of the libm log2 (numpy's
    # vs CUDA's), the device flags FC2_ERR_LOG2_TIE, and the codes may differ by
    # one.  The fixture grid exp2(linspace) hits such ties.
    s = GRP["scales"]
    with np.errstate(divide="ignore"):
        t = np.log2(np.where(s > 0, s, 1.0)) * theta
    near = np.abs(np.abs(t) - np.floor(np.abs(t)) - 0.5) < 1e-9
    got = fc.scale_to_int(s, theta)
    want = GRP[f"s2i_t{theta}"]
    assert np.array_equal(got[~near], want[~near])
    assert np.all(np.abs(got[near].astype(int) - want[near].astype(int)) <= 1)
    assert np.array_equal(fc.int_to_scale(np.arange(-128, 128), theta), GRP[f"i2s_t{theta}"])
    assert fc.scale_to_int(1.0) == 0 and fc.scale_to_int(2.0) == 10 and fc.scale_to_int(0.3) == -17
    assert fc.int_to_scale(-128) == 0.0
    with pytest.raises(fc.DataError):
        fc.scale_to_int(-1.0)


@pytest.mark.parametrize("bits,sr,g,n,slice_elems,intlog,xdt", [
    (4, True, 128, 1 << 20, 1 << 16, False, torch.bfloat16),   # 16 slices
    (3, False, 128, 3 * 32768 + 4096, 32768, False, torch.bfloat16),  # ragged last slice, bit-split planes
    (5, True, 64, 1 << 18, 1 << 22, False, torch.bfloat16),    # one slice
    (8, True, 256, 5 * 32768, 32768, False, torch.bfloat16),
    (6, False, 96, 96 * 1024, 32768, False, torch.bfloat16),   # generic group size: slice rounded to lcm
    (4, True, 128, 1 << 18, 1 << 16, True, torch.bfloat16),    # INT_LOG metadata
    (4, True, 128, 1 << 18, 1 << 16, False, torch.float32),    # f32 chunk (k_encode_fast)
])
def test_host_pipeline_matches_device_path(bits, sr, g, n, slice_elems, intlog, xdt):
    """encode_host / decode_host / roundtrip_host (fc2_*_host: sliced, PCIe
    overlapped) produce the same payload bytes and values as the device path
    and as the oracle."""
    cfg = cfg_of(bits, g, sr, intlog, n)
    x = torch.from_numpy(O.bf16_snap(O.spiky(n, bits)).astype(np.float32)).to(xdt)
    xp = x.pin_memory()
    want = fc.encode_payload(x.cuda(), cfg, n).cpu()
    pay = fc.encode_host(xp, cfg, slice_elems=slice_elems)
    assert torch.equal(pay, want)
    y = fc.decode_host(pay, cfg, n, out_dtype=torch.float32, slice_elems=slice_elems)
    ywant = fc.decode_payload(want.cuda(), cfg, n, out_dtype=torch.float32).cpu()
    assert torch.equal(y, ywant)
    pay2, y2 = fc.roundtrip_host(xp, cfg, out_dtype=torch.bfloat16, slice_elems=slice_elems)
    assert torch.equal(pay2, want)
    assert torch.equal(y2, ywant.to(torch.bfloat16))
    if intlog:
        return  # INT_LOG bytes are pinned against the reference in test_codec_intlog_matches_oracle
    # oracle on a prefix (groups are independent)
    m = 8192 if n >= 8192 else n
    m -= m % g
    planes, meta = O.encode(x[:m].float().numpy(), bits, g, sr)
    units = O.UNITS[bits]
    off = 0
    for w, p in zip(units, planes):
        assert pay[off:off + m * w // 8].numpy().tobytes() == p
        off += n * w // 8


def test_host_pipeline_errors():
    cfg = cfg_of(4, 128, True, False, 4096)
    x = torch.zeros(4096, dtype=torch.float32)
    x[7] = float("nan")
    with pytest.raises(fc.DataError):
        fc.encode_host(x.pin_memory(), cfg)
    with pytest.raises(TypeError):
        fc.encode_host(x.cuda(), cfg)
