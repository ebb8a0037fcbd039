"""Full-size parity at the BASELINE configurations (no sampled slices).

* configs[1]: the whole 64 MiB bf16 tensor (33,554,432 elements), every cell
  of the bit-width sweep (b 2/3/4/5/6/8 x RTN/SR, g128): the complete packed
  payload and the complete decoded output equal the oracle's bytes.
* configs[2]: the Llama-3-8B TP=8 AllReduce (8 ranks x 8192 x 4096 bf16) at
  4-bit and 3-bit SR: ``two_step_allreduce_q`` equals the oracle's two-step
  (collectives.py:263-315) on every element.

The oracle runs with one process per shard / slice (groups are independent,
codec.py:485; shards are independent, collectives.py:276), which keeps these
tests at about a minute each on the GPU box host.
"""

import multiprocessing as mp

import numpy as np
import pytest
import torch

import paper_2508_03760_b200 as fc
from oracle import fc2_oracle as O

pytestmark = pytest.mark.gpu

N_FULL = 8192 * 4096
G = 128


def spiky_bf16_host(n, seed):
    """The bench's synthetic spiky bf16 tensor (N(0,1), 1/64 at +-50), as float32."""
    gen = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(n, device="cuda", generator=gen)
    spike = torch.rand(n, device="cuda", generator=gen) < 1 / 64
    return torch.where(spike, torch.sign(x) * 50, x).to(torch.bfloat16)


_X = None
_RANKS = None


def _enc_slice(job):
    a, b, bits, sr = job
    planes, meta = O.encode(_X[a:b], bits, G, sr)
    dec = O.decode(planes, meta, b - a, bits, G, sr).astype(np.float32)
    return a, planes, meta, dec


def _pool(n):
    return mp.get_context("fork").Pool(max(1, min(n, mp.cpu_count())))


@pytest.mark.parametrize("bits", [2, 3, 4, 5, 6, 8])
@pytest.mark.parametrize("sr", [False, True])
def test_configs1_full_payload_and_decode(bits, sr):
    global _X
    xd = spiky_bf16_host(N_FULL, 100 + bits)
    cfg = fc.QuantConfig(bits, group_size=G, scheme=fc.Scheme.SPIKE_RESERVING if sr else fc.Scheme.RTN,
                         chunk_size=N_FULL)
    pay = fc.encode_payload(xd, cfg, N_FULL).cpu().numpy()
    y32 = fc.decode_payload(torch.from_numpy(pay).cuda(), cfg, N_FULL, out_dtype=torch.float32).cpu().numpy()
    ybf = fc.decode_payload(torch.from_numpy(pay).cuda(), cfg, N_FULL, out_dtype=torch.bfloat16)
    _X = xd.float().cpu().numpy()
    # oracle over 16 group-aligned slices; the full-chunk payload is the
    # concatenation, plane by plane, of the slice payloads (planes are
    # group-contiguous, metadata records are in group order)
    k = 16
    step = N_FULL // k
    with _pool(k) as pool:
        parts = pool.map(_enc_slice, [(a, a + step, bits, sr) for a in range(0, N_FULL, step)])
    parts.sort(key=lambda p: p[0])
    want = b"".join(b"".join(p[1][u] for p in parts) for u in range(len(O.UNITS[bits])))
    want += b"".join(p[2] for p in parts)
    assert len(want) == fc.footprint_bytes(cfg, N_FULL) == pay.size
    assert pay.tobytes() == want
    want_dec = np.concatenate([p[3] for p in parts])
    assert np.array_equal(y32, want_dec)
    assert np.array_equal(ybf.float().cpu().numpy(), O.bf16_snap(want_dec))


def _shard_job(job):
    shard, S, bits, sr = job
    acc = np.zeros(S, dtype=np.float32)
    for src in range(len(_RANKS)):
        acc += O.qdq_f32(_RANKS[src][shard * S:(shard + 1) * S], bits, G, sr)[0]
    return shard, O.qdq_f32(acc, bits, G, sr)[0]


@pytest.mark.parametrize("bits", [4, 3])
def test_configs2_two_step_full_size_bit_exact(bits):
    """8 x (8192 x 4096) bf16, b{4,3} SR g128: every output element equals the
    oracle two-step (one process per shard: the same arithmetic as
    oracle.two_step, which tests/test_oracle_golden.py pins to the reference)."""
    global _RANKS
    N = 8
    xs = [spiky_bf16_host(N_FULL, 1000 + r) for r in range(N)]
    cfg = fc.QuantConfig(bits, group_size=G, scheme=fc.Scheme.SPIKE_RESERVING, chunk_size=G)
    res = fc.two_step_allreduce_q(xs, fc.preset("B200", N), cfg)
    got = res.outputs[0].cpu().numpy()
    for o in res.outputs[1:]:
        assert torch.equal(o, res.outputs[0])
    _RANKS = [x.float().cpu().numpy() for x in xs]
    S = N_FULL // N
    with _pool(N) as pool:
        shards = dict(pool.map(_shard_job, [(j, S, bits, True) for j in range(N)]))
    want = O.bf16_snap(np.concatenate([shards[j] for j in range(N)]))
    assert np.array_equal(got, want)
    # the oracle's own two-step agrees on a leading slice (pins the pooled form)
    m = N * G * 64
    w2, _ = O.two_step([r[:m] for r in _RANKS], bits, G, True)
    two = fc.two_step_allreduce_q([x[:m] for x in xs], fc.preset("B200", N), cfg).outputs[0].cpu().numpy()
    assert np.array_equal(two, w2[0])
