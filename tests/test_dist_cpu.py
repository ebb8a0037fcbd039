"""Multi-rank host logic of the SPMD path on CPU: world_size 2 and 3 over gloo.

The transport-agnostic orchestration (``dist.two_step_via_collectives``) is
driven with a test-only codec double built on the oracle, so the exchange
plan (shard geometry, padding, slot layout, which rank sends what where, the
rank-order reduction) is checked bit-for-bit against the reference algorithm
without a GPU.  The product codec is the CUDA library (tests/test_dist_gpu.py).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2508_03760_b200 as fc
from oracle import fc2_oracle as O
from paper_2508_03760_b200.dist import TwoStepLayout, a2a_slot_offsets, two_step_via_collectives


class OracleCodec:
    """Test double of dist.CudaCodec: same interface, numpy oracle inside."""

    def __init__(self, cfg):
        self.cfg = cfg

    def _enc(self, v):
        c = self.cfg
        planes, meta = O.encode(v, c.bitwidth, c.group_size, c.spike_reserving)
        return np.frombuffer(b"".join(planes) + meta, dtype=np.uint8)

    def _dec(self, buf, n):
        c = self.cfg
        raw = bytes(buf)
        planes, pos = [], 0
        for w in O.UNITS[c.bitwidth]:
            planes.append(raw[pos:pos + n * w // 8])
            pos += n * w // 8
        meta = raw[pos:pos + (n // c.group_size) * O.record_nbytes(c.spike_reserving, False)]
        return O.decode(planes, meta, n, c.bitwidth, c.group_size, c.spike_reserving).astype(np.float32)

    def empty(self, nbytes):
        return torch.zeros(nbytes, dtype=torch.uint8)

    def encode_shards(self, x, lay, send):
        xs = x.numpy()
        for j in range(lay.world):
            blk = np.zeros(lay.shard_len, np.float32)
            v = lay.valid(j)
            blk[:v] = xs[j * lay.shard_len: j * lay.shard_len + v]
            b = self._enc(blk)
            send[j * lay.slot_bytes: j * lay.slot_bytes + b.size] = torch.from_numpy(b.copy())

    def reduce(self, recv, lay, out):
        acc = np.zeros(lay.shard_len, np.float32)
        for s in range(lay.world):
            acc += self._dec(recv[s * lay.slot_bytes:(s + 1) * lay.slot_bytes].numpy(), lay.shard_len)
        b = self._enc(acc)
        out[:b.size] = torch.from_numpy(b.copy())

    def decode_gathered(self, gath, lay, y):
        parts = [self._dec(gath[o * lay.slot_bytes:(o + 1) * lay.slot_bytes].numpy(), lay.shard_len)
                 for o in range(lay.world)]
        y.copy_(torch.from_numpy(O.bf16_snap(np.concatenate(parts)[:lay.n])))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, bits, g, sr, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = fc.QuantConfig(bits, group_size=g, scheme=fc.Scheme.SPIKE_RESERVING if sr else fc.Scheme.RTN,
                             chunk_size=g)
        seeds = O.child_seeds(seed, world)
        x = torch.from_numpy(O.bf16_snap(O.spiky(n, seeds[rank])).astype(np.float32))
        lay = TwoStepLayout.make(n, world, cfg)
        y = two_step_via_collectives(x, OracleCodec(cfg), lay)
        q.put((rank, y.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,bits,g,sr", [(2, 5000, 4, 128, True), (3, 4096, 3, 32, False),
                                               (2, 1024, 8, 128, True)])
def test_two_step_orchestration_matches_reference_algorithm(world, n, bits, g, sr):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, bits, g, sr, 7, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    payloads = [O.bf16_snap(O.spiky(n, s)).astype(np.float32) for s in O.child_seeds(7, world)]
    want, _ = O.two_step(payloads, bits, g, sr)
    for r in range(world):
        assert np.array_equal(np.frombuffer(got[r], dtype=np.float32), want[0])


def test_layout_matches_reference_padding():
    cfg = fc.QuantConfig(4, group_size=128, scheme=fc.Scheme.SPIKE_RESERVING)
    lay = TwoStepLayout.make(5000, 8, cfg)
    assert lay.padded == 8 * 128 * 5 and lay.shard_len == 640  # collectives.py:275-276
    assert [lay.valid(j) for j in range(8)] == [640] * 7 + [520]
    assert lay.shard_bytes == fc.footprint_bytes(cfg, 640) and lay.slot_bytes % 16 == 0
    big = TwoStepLayout.make(8192 * 4096, 8, cfg)
    assert big.shard_len == 4194304 and big.shard_bytes == 2490368


def test_a2a_slot_offsets_are_prefix_sums():
    cfg = fc.QuantConfig(4, group_size=128)
    m = np.array([[5, 300, 0], [129, 0, 7], [0, 256, 3]])
    offs = a2a_slot_offsets(m, cfg, dst=1)
    f = lambda k: -(-fc.footprint_bytes(cfg, -(-k // 128) * 128) // 16) * 16
    assert offs == [0, f(300), f(300), f(300) + f(256)]
