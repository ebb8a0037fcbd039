"""MoE token dispatch / combine (BASELINE configs[3]) against
the oracle's restatement: the reference block All2All (collectives.py:428-482)
on the routed token rows, then the rank-order fp32 combine.

Bit-exact: the received rows (float32) and the combined outputs equal the
oracle's on every element, including the full DeepSeek-V3-like shape
(4096 tokens x 7168 hidden, top-8 of 256 experts, EP = 8)."""

import hashlib
import multiprocessing as mp

import numpy as np
import pytest
import torch

import paper_2508_03760_b200 as fc
from oracle import fc2_oracle as O

pytestmark = pytest.mark.gpu


def cfg(bits, g, sr):
    return fc.QuantConfig(bits, group_size=g, scheme=fc.Scheme.SPIKE_RESERVING if sr else fc.Scheme.RTN,
                          chunk_size=g)


def routing(T, K, E, seed):
    """K distinct experts per token, uniformly at random."""
    rng = np.random.default_rng(seed)
    return np.argsort(rng.random((T, E)), axis=1)[:, :K].astype(np.int64)


def tokens_bf16(T, H, seed):
    return O.bf16_snap(O.spiky(T * H, seed)).astype(np.float32).reshape(T, H)


@pytest.mark.parametrize("N,Ts,H,K,E,bits,g,sr", [
    (4, [100, 37, 64, 5], 256, 4, 16, 4, 128, True),
    (2, [33, 64], 1024, 2, 8, 3, 32, False),
    (3, [17, 0, 50], 384, 3, 6, 5, 64, True),
    (8, [64] * 8, 7168, 8, 256, 4, 128, True),
    (2, [20, 30], 264, 2, 8, 4, 24, True),  # generic encoder (g = 24) + unfused combine (H % 32 != 0)
    (2, [40, 9], 1024, 2, 8, 6, 32, False),
    (2, [40, 25], 1024, 2, 8, 8, 128, True),  # b8 SR: per-quad reserved-value substitution in the combine
])
@pytest.mark.parametrize("resident", ["host_f32", "cuda_bf16"])
def test_moe_dispatch_combine_match_oracle(N, Ts, H, K, E, bits, g, sr, resident):
    toks = [tokens_bf16(T, H, 10 + s) for s, T in enumerate(Ts)]
    ids = [routing(T, K, E, 50 + s) for s, T in enumerate(Ts)]
    c = cfg(bits, g, sr)
    topo = fc.preset("B200", N)
    xin = toks if resident == "host_f32" else [torch.from_numpy(t).cuda().to(torch.bfloat16) for t in toks]
    res = fc.moe_dispatch_q(xin, ids, topo, c, n_experts=E)
    want, routes = O.moe_dispatch(toks, ids, bits, g, sr, E)
    for d in range(N):
        assert np.array_equal(res.outputs[d].cpu().numpy(), want[d])
    lay = res.layout
    for s in range(N):
        for d in range(N):
            assert lay.counts[s, d] == routes[s][0][d].size
    # expert outputs: any function of the received rows (here a scaled copy, bf16)
    yo = [O.bf16_snap(w * 0.5 + 1.0).astype(np.float32) for w in want]
    yin = yo if resident == "host_f32" else [torch.from_numpy(y).cuda().to(torch.bfloat16) for y in yo]
    back = fc.moe_combine_q(yin, lay, topo, c)
    want_c = O.moe_combine(yo, routes, bits, g, sr)
    for s in range(N):
        assert np.array_equal(back.outputs[s].cpu().numpy(), want_c[s])
    # ledger: one transfer per remote non-empty block, packed bytes of that block
    nblk = sum(1 for s in range(N) for d in range(N) if s != d and lay.counts[s, d])
    assert len(res.ledger.events) == nblk and len(back.ledger.events) == nblk


def test_moe_errors():
    topo = fc.preset("B200", 2)
    c = cfg(4, 128, True)
    toks = [tokens_bf16(8, 256, s) for s in range(2)]
    bad = [routing(8, 2, 8, 0), routing(8, 2, 8, 1)]
    bad[1][3, 1] = 8  # expert id out of range
    with pytest.raises(fc.ConfigError):
        fc.moe_dispatch_q(toks, bad, topo, c, n_experts=8)
    with pytest.raises(fc.ConfigError):  # hidden not a multiple of 8
        fc.moe_dispatch_q([t[:, :100] for t in toks], [routing(8, 2, 8, 0)] * 2, topo, c, n_experts=8)
    ids = [routing(8, 2, 8, 0), routing(8, 2, 8, 1)]
    nan = [t.copy() for t in toks]
    nan[0][2, 5] = np.nan  # a token row that routes somewhere
    with pytest.raises(fc.DataError):
        fc.moe_dispatch_q(nan, ids, topo, c, n_experts=8)


# ---- full configs[3] shape: 8 ranks x 4096 tokens x 7168, top-8 of 256 ----

_TOK = None
_ROUTES = None
_YO = None


def _dispatch_block_hash(job):
    s, d, bits, g, sr = job
    rows = _ROUTES[s][0][d]
    blk = _TOK[s][rows].reshape(-1)
    if s != d and blk.size:
        plen = -(-blk.size // g) * g
        blk = O.qdq_f32(np.pad(blk, (0, plen - blk.size)), bits, g, sr)[0][:blk.size]
    return (s, d), hashlib.sha256(np.ascontiguousarray(blk, dtype=np.float32).tobytes()).hexdigest()


def _combine_hash(job):
    s, bits, g, sr, counts = job
    N = len(_YO)
    H = _YO[0].shape[1]
    acc = np.zeros((_ROUTES[s][1].shape[0], H), dtype=np.float32)
    for e in range(N):
        r0 = int(counts[:s, e].sum())
        k = int(counts[s, e])
        rows = _YO[e][r0:r0 + k].reshape(-1)
        if e != s and rows.size:
            plen = -(-rows.size // g) * g
            rows = O.qdq_f32(np.pad(rows, (0, plen - rows.size)), bits, g, sr)[0][:rows.size]
        sel = _ROUTES[s][0][e]
        acc[sel] = acc[sel] + rows.reshape(-1, H)
    return s, hashlib.sha256(acc.tobytes()).hexdigest()


def test_moe_configs3_full_shape_bit_exact():
    global _TOK, _ROUTES, _YO
    N, T, H, K, E, bits, g, sr = 8, 4096, 7168, 8, 256, 4, 128, True
    c = cfg(bits, g, sr)
    topo = fc.preset("B200", N)
    gen = torch.Generator(device="cuda").manual_seed(3)
    xs = []
    for s in range(N):
        x = torch.randn(T * H, device="cuda", generator=gen)
        spike = torch.rand(T * H, device="cuda", generator=gen) < 1 / 64
        xs.append(torch.where(spike, torch.sign(x) * 50, x).to(torch.bfloat16).reshape(T, H))
    ids = [routing(T, K, E, 900 + s) for s in range(N)]
    res = fc.moe_dispatch_q(xs, ids, topo, c, n_experts=E)
    lay = res.layout
    _TOK = [x.float().cpu().numpy() for x in xs]
    _ROUTES = [O.moe_route(i, N, E) for i in ids]
    for s in range(N):
        for d in range(N):
            assert lay.counts[s, d] == _ROUTES[s][0][d].size
    got = {}
    for d in range(N):
        out = res.outputs[d]
        off = 0
        for s in range(N):
            k = int(lay.counts[s, d])
            got[(s, d)] = hashlib.sha256(out[off:off + k].cpu().numpy().tobytes()).hexdigest()
            off += k
    with mp.get_context("fork").Pool(min(16, mp.cpu_count())) as pool:
        want = dict(pool.map(_dispatch_block_hash, [(s, d, bits, g, sr) for s in range(N) for d in range(N)]))
    assert got == want
    # combine of bf16 expert outputs (a scaled copy of the received rows)
    ys = [(o * 0.5 + 1.0).to(torch.bfloat16) for o in res.outputs]
    del res
    back = fc.moe_combine_q(ys, lay, topo, c)
    _YO = [y.float().cpu().numpy() for y in ys]
    got_c = {s: hashlib.sha256(back.outputs[s].cpu().numpy().tobytes()).hexdigest() for s in range(N)}
    with mp.get_context("fork").Pool(min(8, mp.cpu_count())) as pool:
        want_c = dict(pool.map(_combine_hash, [(s, bits, g, sr, lay.counts) for s in range(N)]))
    assert got_c == want_c
