"""GPU parity of the quantized collectives against the reference's own outputs
(tests/golden/*.npz) and the pinned oracle."""

import numpy as np
import pytest
import torch

import paper_2508_03760_b200 as fc
from oracle import fc2_oracle as O
from tests.golden_io import load

pytestmark = pytest.mark.gpu

TS, TS_IDX = load("two_step_golden.npz")
A2A, A2A_IDX = load("a2a_golden.npz")


def cfg(bits, g, sr):
    return fc.QuantConfig(bits, group_size=g, scheme=fc.Scheme.SPIKE_RESERVING if sr else fc.Scheme.RTN,
                          chunk_size=g)


@pytest.mark.parametrize("case", [c for c in TS_IDX if c["key"] != "ts_identical"], ids=lambda c: c["key"])
@pytest.mark.parametrize("resident", ["host", "cuda_f32", "cuda_bf16"])
def test_two_step_matches_reference(case, resident):
    payloads = list(TS["in_" + case["key"]])
    if resident == "cuda_f32":
        payloads = [torch.from_numpy(p).cuda() for p in payloads]
    elif resident == "cuda_bf16":
        payloads = [torch.from_numpy(p).cuda().to(torch.bfloat16) for p in payloads]
    topo = fc.preset("H800", case["N"])
    res = fc.two_step_allreduce_q(payloads, topo, cfg(case["bits"], case["g"], case["sr"]))
    want = TS["out_" + case["key"]]
    outs = [o.cpu().numpy() if isinstance(o, torch.Tensor) else o for o in res.outputs]
    for o in outs:
        assert np.array_equal(o, want)
    rep = fc.volume_report(res.ledger, topo)
    assert rep["total_raw"] == case["total_raw"] and rep["total_actual"] == case["total_actual"]
    assert len(res.ledger.events) == case["events"]


def test_two_step_identical_payloads_fold():
    p = TS["in_ts_identical"]
    res = fc.two_step_allreduce_q([p.copy() for _ in range(8)], fc.preset("B200"), fc.QuantConfig(5))
    assert np.array_equal(res.outputs[0], TS["out_ts_identical"])


@pytest.mark.parametrize("N,n,bits,g,sr", [(8, 1 << 16, 4, 128, True), (8, 100003, 3, 128, True),
                                          (4, 1 << 15, 2, 32, True), (2, 77777, 6, 64, False),
                                          (8, 40960, 5, 40, True), (16, 1 << 14, 4, 128, True)])
def test_two_step_matches_oracle(N, n, bits, g, sr):
    payloads = [O.bf16_snap(O.spiky(n, s)).astype(np.float32) for s in O.child_seeds(n, N)]
    res = fc.two_step_allreduce_q(payloads, fc.preset("B200", N), cfg(bits, g, sr))
    want, _ = O.two_step(payloads, bits, g, sr)
    assert np.array_equal(res.outputs[0], want[0])


@pytest.mark.parametrize("N,bits,g,sr", [(8, 4, 128, True), (4, 3, 64, True), (8, 8, 128, True), (2, 2, 32, False),
                                         (4, 4, 64, True), (3, 8, 32, True)])
def test_two_step_stress_matches_oracle(N, bits, g, sr):
    """The stage-2 reducer on the stress mix (tests/test_gpu_codec.py): sums of
    groups from different regimes across ranks, requantized."""
    from tests.test_gpu_codec import stress

    n = N * g * 2048  # the fast stage-2 shape (1024-element tiles, 16-byte aligned slots)
    payloads = [stress(n, 500 + r, g) for r in range(N)]
    res = fc.two_step_allreduce_q(payloads, fc.preset("B200", N), cfg(bits, g, sr))
    want, _ = O.two_step(payloads, bits, g, sr)
    assert np.array_equal(res.outputs[0], want[0])


def test_two_step_nonfinite_raises():
    payloads = [np.ones(4096, np.float32) for _ in range(4)]
    payloads[2][100] = np.nan
    with pytest.raises(fc.DataError):
        fc.two_step_allreduce_q(payloads, fc.preset("B200", 4), fc.QuantConfig(4))


def test_two_step_error_bound_full_size():
    """Llama TP=8 shape (8192 x 4096 bf16 per rank, 4-bit SR g128): max abs
    error vs the exact sum <= sum over ranks of one quantization step per rank
    contribution plus one step of the reduced shard (north-star tolerance);
    the relative L2 error is reported."""
    N, n = 8, 8192 * 4096
    gen = torch.Generator(device="cuda").manual_seed(0)
    xs = []
    for _ in range(N):
        x = torch.randn(n, device="cuda", generator=gen)
        spike = torch.rand(n, device="cuda", generator=gen) < 1 / 64
        xs.append(torch.where(spike, torch.sign(x) * 50, x).to(torch.bfloat16))
    c = cfg(4, 128, True)
    res = fc.two_step_allreduce_q(xs, fc.preset("B200"), c)
    exact = torch.zeros(n, dtype=torch.float64, device="cuda")
    for x in xs:
        exact += x.double()
    out = res.outputs[0].double()
    err = (out - exact).abs()
    # per-group step of each rank's contribution and of the reduced sum
    def step(v):
        r = v.view(-1, 128)
        s = torch.sort(r, dim=1).values
        return ((s[:, -2] - s[:, 1]) / 15.0).repeat_interleave(128)
    bound = sum(step(x.double()) for x in xs) + step(exact) + exact.abs() * 2.0 ** -8 + 1e-6
    spikes_ok = err <= bound
    rel_l2 = float(torch.linalg.norm(out - exact) / torch.linalg.norm(exact))
    print(f"two-step 8x64MiB b4 SR: max abs err {float(err.max()):.4g}, rel-L2 {rel_l2:.4g}")
    assert bool(spikes_ok.all())
    assert rel_l2 < 0.3


@pytest.mark.parametrize("case", A2A_IDX, ids=lambda c: c["key"])
@pytest.mark.parametrize("resident", ["host", "cuda"])
def test_a2a_dispatch_matches_reference(case, resident):
    key, N = case["key"], case["N"]
    payloads = [A2A[f"in_{key}_{i}"] for i in range(N)]
    if resident == "cuda":
        payloads = [torch.from_numpy(p).cuda() for p in payloads]
    mat = A2A[f"matrix_{key}"] if case["matrix"] else None
    topo = fc.preset("H800")
    res = fc.all2all_dispatch_q(payloads, topo, cfg(case["bits"], case["g"], case["sr"]), mat)
    flat = np.concatenate([np.asarray(res.outputs[d][s].cpu() if isinstance(res.outputs[d][s], torch.Tensor)
                                      else res.outputs[d][s]) for d in range(N) for s in range(N)])
    assert np.array_equal(flat, A2A["out_" + key])
    rep = fc.volume_report(res.ledger, topo)
    assert rep["total_raw"] == case["total_raw"] and rep["total_actual"] == case["total_actual"]


def test_a2a_combine_matches_oracle():
    N = 8
    rng = np.random.default_rng(4)
    blocks = [[O.bf16_snap(rng.normal(0, 1, int(rng.integers(0, 3)) * 7168)).astype(np.float32)
               for _ in range(N)] for _ in range(N)]
    res = fc.all2all_combine_q(blocks, fc.preset("B200"), cfg(4, 128, True))
    want = O.a2a_combine(blocks, 4, 128, True)
    for d in range(N):
        for s in range(N):
            assert np.array_equal(res.outputs[d][s], want[d][s])


def test_a2a_zero_matrix_and_shape_errors():
    N = 8
    topo = fc.preset("B200")
    res = fc.all2all_dispatch_q([np.zeros(0, np.float32)] * N, topo, fc.QuantConfig(8),
                                np.zeros((N, N), dtype=int))
    assert res.ledger.total_raw == 0
    with pytest.raises(fc.ConfigError):
        fc.all2all_dispatch_q([np.zeros(64, np.float32)] * N, topo, fc.QuantConfig(8), np.zeros((3, 3), int))


@pytest.mark.parametrize("bits,g,sr,S,stride_pad", [(4, 128, True, 8192, 0), (3, 64, False, 4096, 16),
                                                    (4, 128, True, 4096, 8), (5, 96, True, 96 * 40, 0)])
def test_reduce_requant_batch_equals_per_shard(bits, g, sr, S, stride_pad):
    """fc2_reduce_requant_batch (the one-shot AllReduce's local reduce of every
    shard) == one fc2_reduce_requant per shard, byte for byte; covers the CTA
    kernel, a stride that only the per-launch reducers take (8-byte aligned),
    and a non-fast group size."""
    import ctypes

    from paper_2508_03760_b200 import _lib
    from paper_2508_03760_b200.collectives import reduce_requant

    c = cfg(bits, g, sr)
    N, K = 4, 3
    F = fc.footprint_bytes(c, S)
    slot = (F + 15) // 16 * 16 + stride_pad
    src = torch.zeros(N * K * slot + 64, dtype=torch.uint8, device="cuda")
    for s in range(N):
        for k in range(K):
            x = torch.from_numpy(O.bf16_snap(O.spiky(S, 100 * s + k)).astype(np.float32)).cuda()
            src[(s * K + k) * slot:(s * K + k) * slot + F] = fc.encode_payload(x, c, S)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    want = torch.zeros(K * slot, dtype=torch.uint8, device="cuda")
    for k in range(K):
        reduce_requant(c, [src.data_ptr() + (s * K + k) * slot for s in range(N)], S,
                       [want.data_ptr() + k * slot], err)
    got = torch.zeros_like(want)
    cs = c.c_struct()
    _lib.check(_lib.lib().fc2_reduce_requant_batch(
        ctypes.byref(cs), N, _lib.ptr_array([src.data_ptr() + s * K * slot for s in range(N)]), S, K, slot, 1,
        _lib.ptr_array([got.data_ptr()]), slot, err.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    for k in range(K):
        assert torch.equal(got[k * slot:k * slot + F], want[k * slot:k * slot + F])


def test_reduce_requant_batch_rejects_bad_shapes():
    import ctypes

    from paper_2508_03760_b200 import _lib

    c = cfg(4, 128, True).c_struct()
    buf = torch.zeros(1 << 16, dtype=torch.uint8, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    ptrs = _lib.ptr_array([buf.data_ptr()])
    # nshard < 1 and a shard that is not a group multiple are ConfigErrors, like fc2_reduce_requant
    with pytest.raises(fc.ConfigError):
        _lib.check(_lib.lib().fc2_reduce_requant_batch(ctypes.byref(c), 1, ptrs, 1024, 0, 0, 1, ptrs, 0,
                                                       err.data_ptr(), st))
    with pytest.raises(fc.ConfigError):
        _lib.check(_lib.lib().fc2_reduce_requant_batch(ctypes.byref(c), 1, ptrs, 1000, 2, 4096, 1, ptrs, 4096,
                                                       err.data_ptr(), st))


def test_host_entry_points_validate_buffers():
    c = cfg(4, 128, True)
    x = torch.zeros(4096, dtype=torch.bfloat16).pin_memory()
    with pytest.raises(TypeError):
        fc.roundtrip_host(x.cuda(), c)
    with pytest.raises(fc.DecodeFormatError):
        fc.decode_host(torch.zeros(16, dtype=torch.uint8).pin_memory(), c, 4096)
    with pytest.raises(fc.ConfigError):
        fc.encode_host(torch.zeros(1000, dtype=torch.bfloat16).pin_memory(), c)  # not a group multiple


HIER, HIER_IDX = load("hier_golden.npz")


@pytest.mark.gpu
@pytest.mark.parametrize("case", HIER_IDX, ids=lambda c: c["key"])
def test_hierarchical_matches_reference(case):
    """hierarchical_two_step_q on the GPU codec == the reference's outputs,
    ledger events and volume report on bridged fabrics (collectives.py:318-425)."""
    import json

    topo = fc.preset("L40") if case["topo"] == "L40" else fc.Topology.from_json(
        json.loads(bytes(HIER["topo_pcie4"]).decode()))
    payloads = list(HIER["in_" + case["key"]])
    c = fc.QuantConfig(case["bits"], group_size=case["g"],
                       scheme=fc.Scheme.SPIKE_RESERVING if case["sr"] else fc.Scheme.RTN)
    res = fc.hierarchical_two_step_q(payloads, topo, c)
    want = HIER["out_" + case["key"]]
    for r in range(case["N"]):
        assert np.array_equal(res.outputs[r], want[r])
    got_ev = [[e.stage, e.wave, e.src, e.dst, e.elements, e.actual_bytes] for e in res.ledger.events]
    assert got_ev == case["events"]
    assert [[s.name, len(s.transfers), len(s.computes)] for s in res.trace.stages] == case["stages"]
    assert fc.volume_report(res.ledger, topo) == case["report"]
    # device-resident payloads give the same values
    dres = fc.hierarchical_two_step_q([torch.from_numpy(p).cuda() for p in payloads], topo, c)
    assert np.array_equal(dres.outputs[0].cpu().numpy(), want[0])
