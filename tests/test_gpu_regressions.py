"""Regression tests for round-1 review findings (ADVICE.md / VERDICT.md)."""

import numpy as np
import pytest
import torch

import paper_2508_03760_b200 as fc
from oracle import fc2_oracle as O
from paper_2508_03760_b200 import fileio

pytestmark = pytest.mark.gpu


def cfg(bits, g, sr, chunk=None):
    return fc.QuantConfig(bits, group_size=g, scheme=fc.Scheme.SPIKE_RESERVING if sr else fc.Scheme.RTN,
                          chunk_size=chunk or g)


@pytest.mark.parametrize("bits", [3, 7, 5])
@pytest.mark.parametrize("n", [96, 32 * 37, 32 * 1001, 64 * 99])
@pytest.mark.parametrize("sr", [False, True])
def test_decode_plane_offsets_not_16_byte_aligned(bits, n, sr):
    """B = 3 / 7 with n % 64 == 32 put the second plane at an 8-byte offset;
    the vectorised decoder must not be used there (it would fault)."""
    x = O.bf16_snap(O.spiky(n, n + bits)).astype(np.float32)
    c = cfg(bits, 32, sr, n)
    chunk = fc.encode_chunk(x, c)
    planes, meta = O.encode(x, bits, 32, sr)
    assert chunk.planes == planes and chunk.meta == meta
    assert np.array_equal(fc.decode_chunk(chunk), O.decode(planes, meta, n, bits, 32, sr))
    pay = torch.from_numpy(np.frombuffer(b"".join(planes) + meta, dtype=np.uint8).copy()).cuda()
    for dt in (torch.float32, torch.bfloat16):
        y = fc.decode_payload(pay, c, n, out_dtype=dt).float().cpu().numpy()
        want = O.decode(planes, meta, n, bits, 32, sr).astype(np.float32)
        assert np.array_equal(y, want if dt == torch.float32 else O.bf16_snap(want))


def test_two_step_odd_shard_b3_default_group():
    """n = 100003 on 8 ranks with QuantConfig(3) (g = 32): shard 12512, 12512 % 64 == 32."""
    payloads = [O.bf16_snap(O.spiky(100003, s)).astype(np.float32) for s in O.child_seeds(77, 8)]
    res = fc.two_step_allreduce_q(payloads, fc.preset("B200"), fc.QuantConfig(3))
    want, _ = O.two_step(payloads, 3, 32, False)
    assert np.array_equal(res.outputs[0], want[0])


def test_all2all_odd_blocks_b7_g32():
    m = np.array([[32 * 3, 32 * 5], [32 * 7, 32]])
    payloads = [O.bf16_snap(O.spiky(int(m[r].sum()), 40 + r)).astype(np.float32) for r in range(2)]
    res = fc.all2all_dispatch_q(payloads, fc.preset("B200", 2), cfg(7, 32, True), dispatch_matrix=m)
    want = O.a2a_dispatch(payloads, 7, 32, True, m)
    for d in range(2):
        for s in range(2):
            assert np.array_equal(res.outputs[d][s], want[d][s])


@pytest.mark.parametrize("bits,g,chunk", [(3, 40, 4080), (5, 24, 96), (3, 40, 40), (4, 24, 4080)])
def test_file_chunks_with_unaligned_footprints(bits, g, chunk):
    """Per-chunk footprints that are not word multiples (e.g. 19 or 1938 bytes)."""
    n = chunk * 3 + g * 5
    x = O.bf16_snap(O.spiky(n, bits * g)).astype(np.float32)
    c = fc.QuantConfig(bits, group_size=g, scheme=fc.Scheme.SPIKE_RESERVING, chunk_size=chunk)
    chunks = fileio.quantize_tensor(x, c)
    pos = 0
    for ch in chunks:
        m = ch.element_count
        planes, meta = O.encode(x[pos:pos + m], bits, g, True)
        assert ch.planes == planes and ch.meta == meta
        pos += m
    assert pos == n
    y = fileio.dequantize_chunks(chunks)
    want = np.concatenate([O.decode(ch.planes, ch.meta, ch.element_count, bits, g, True) for ch in chunks])
    assert np.array_equal(y, want)
    dchunks = fileio.quantize_tensor(torch.from_numpy(x).cuda(), c, device_payload=True)
    assert b"".join(ch.to_bytes() for ch in dchunks) == b"".join(ch.to_bytes() for ch in chunks)


@pytest.mark.parametrize("where", [(0, 0), (1, 1), (0, 1)])
def test_all2all_nonfinite_anywhere_raises(where):
    """collectives.py:152-164 rejects NaN/inf in any block, the diagonal included."""
    N = 2
    payloads = [np.ones(256, np.float32) for _ in range(N)]
    src, dst = where
    payloads[src][dst * 128 + 5] = np.nan
    with pytest.raises(fc.DataError):
        fc.all2all_dispatch_q(payloads, fc.preset("B200", N), cfg(4, 128, True))
    blocks = [[np.ones(128, np.float32) for _ in range(N)] for _ in range(N)]
    blocks[src][dst][3] = np.inf
    with pytest.raises(fc.DataError):
        fc.all2all_combine_q(blocks, fc.preset("B200", N), cfg(4, 128, True))


def test_payload_buffer_validation():
    """Caller-provided buffers that are too small, of the wrong dtype or
    non-contiguous raise ConfigError instead of being overrun."""
    cfg = fc.QuantConfig(4, group_size=128, chunk_size=128)
    x = torch.zeros(1024, dtype=torch.bfloat16, device="cuda")
    F = fc.footprint_bytes(cfg, 1024)
    with pytest.raises(fc.ConfigError):
        fc.encode_payload(x, cfg, 1024, out=torch.empty(F - 1, dtype=torch.uint8, device="cuda"))
    with pytest.raises(fc.ConfigError):
        fc.encode_payload(x, cfg, 1024, out=torch.empty(F, dtype=torch.int32, device="cuda"))
    with pytest.raises(fc.ConfigError):
        fc.encode_payload(x, cfg, 512)
    pay = fc.encode_payload(x, cfg, 1024)
    with pytest.raises(fc.ConfigError):
        fc.decode_payload(pay[:-1], cfg, 1024)
    with pytest.raises(fc.ConfigError):
        fc.decode_payload(pay, cfg, 1024, out=torch.empty(1023, device="cuda"))
    with pytest.raises(fc.ConfigError):
        fc.decode_payload(pay, cfg, 1024, out=torch.empty(2048, device="cuda")[::2])
