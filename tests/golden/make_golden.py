"""Generate golden fixtures by running the REAL reference (build container only).

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

The reference (``qcomm`` under /root/reference/pkg/src, pure Python+numpy) is
imported read-only; nothing here is copied into the product.  The fixtures
hold the inputs plus the reference's own outputs, so the GPU box (which has no
/root/reference) can check both the oracle and the CUDA path against them.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from dataclasses import replace
from pathlib import Path

sys.dont_write_bytecode = True
REF = Path(os.environ.get("FC2_REFERENCE", "/root/reference/pkg/src"))
sys.path.insert(0, str(REF))

import numpy as np  # noqa: E402
import qcomm  # noqa: E402
from qcomm import (  # noqa: E402
    QuantConfig,
    ScaleEncoding,
    Scheme,
    all2all_dispatch_q,
    bf16_round,
    decode_chunk,
    default_spiky_spec,
    encode_chunk,
    gen_synthetic,
    preset,
    rank_seeds,
    two_step_allreduce_q,
    volume_report,
)

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def edge_inputs(g_max: int = 128) -> np.ndarray:
    """Hand-built groups that stress the arithmetic contract."""
    rows = []
    rng = np.random.default_rng(1234)

    def grp(vals):
        vals = np.asarray(vals, dtype=np.float64)
        assert vals.size == g_max
        rows.append(vals)

    grp(np.full(g_max, 5.0))                                   # constant
    grp(np.zeros(g_max))                                       # all zero
    grp(np.tile([0.0, 0.5, 2.5, 3.0], g_max // 4))             # exact .5 ties
    grp(np.arange(g_max, dtype=np.float64) / 4.0)              # regular grid, ties at many bits
    v = rng.normal(0, 1, g_max); v[0] = -40; v[1] = 40; grp(v)  # spikes at slots 0/1
    v = rng.normal(0, 1, g_max); v[-1] = -40; v[-2] = 40; grp(v)  # spikes at the end
    v = rng.normal(0, 1, g_max); v[[3, 9]] = -7.0; v[[5, 77]] = 9.0; grp(v)  # duplicate extremes
    grp(np.float32(1e-38) * rng.integers(1, 5, g_max))         # tiny (subnormal-ish) range
    grp(rng.normal(0, 1, g_max) * 3e37)                        # huge values
    grp(1000.0 + rng.integers(0, 16, g_max) / 16.0)            # large offset, small range
    v = np.full(g_max, 2.0); v[17] = 1.0; grp(v)               # single low outlier
    v = np.full(g_max, 2.0); v[17] = 3.0; grp(v)               # single high outlier
    grp(-np.arange(g_max, dtype=np.float64))                   # strictly decreasing
    grp(np.tile([1.0, -1.0], g_max // 2))                      # two values
    v = rng.normal(0, 1, g_max); grp(v)
    grp(np.linspace(-1, 1, g_max))
    return bf16_round(np.concatenate(rows)).astype(np.float32)


def codec_fixture():
    inputs = {
        "spiky_bf16": bf16_round(gen_synthetic(default_spiky_spec(4096, 1))).astype(np.float32),
        "normal_f64": np.random.default_rng(7).normal(0, 3, 4096) * np.random.default_rng(8).uniform(0.01, 100, 4096),
        "edge_bf16": edge_inputs(128),
    }
    arrays = {f"in_{k}": v for k, v in inputs.items()}
    cases = []
    for name, vals in inputs.items():
        for bits in range(2, 9):
            for g in (8, 32, 128):
                for sch in (Scheme.RTN, Scheme.SPIKE_RESERVING):
                    for enc in (ScaleEncoding.BF16, ScaleEncoding.INT_LOG):
                        if name == "normal_f64" and g == 8:
                            continue
                        cfg = QuantConfig(bits, group_size=g, scheme=sch, scale_encoding=enc,
                                          chunk_size=vals.size)
                        ch = encode_chunk(vals, cfg)
                        key = f"{name}_b{bits}_g{g}_{sch.value}_{enc.value}"
                        payload = np.frombuffer(b"".join(ch.planes) + ch.meta, dtype=np.uint8)
                        arrays[f"payload_{key}"] = payload
                        dec = decode_chunk(ch)
                        cases.append(dict(key=key, input=f"in_{name}", bits=bits, g=g,
                                          sr=sch is Scheme.SPIKE_RESERVING,
                                          intlog=enc is ScaleEncoding.INT_LOG,
                                          planes=[len(p) for p in ch.planes],
                                          meta=len(ch.meta), decoded_sha=sha(dec),
                                          decoded_f32_sha=sha(dec.astype(np.float32))))
    arrays["index"] = np.frombuffer(json.dumps(cases).encode(), dtype=np.uint8)
    np.savez_compressed(OUT / "codec_golden.npz", **arrays)
    return len(cases)


def make_topo(n):
    base = preset("H800")
    return qcomm.Topology(name=f"nv{n}", devices=base.devices[:n], links=base.links[:n])


def two_step_fixture():
    cases = [
        # (N, n, bits, g, sr, seed)
        (8, 16384, 4, 128, True, 0),
        (8, 5000, 3, 128, True, 1),
        (4, 8192, 2, 32, False, 2),
        (2, 4096, 8, 128, True, 3),
        (8, 16384, 4, 128, False, 4),
        (8, 8192, 2, 32, True, 5),
        (3, 3000, 5, 64, True, 6),
        (1, 1024, 4, 128, True, 7),
    ]
    arrays, index = {}, []
    for N, n, bits, g, sr, seed in cases:
        cfg = QuantConfig(bits, group_size=g,
                          scheme=Scheme.SPIKE_RESERVING if sr else Scheme.RTN)
        payloads = [bf16_round(gen_synthetic(default_spiky_spec(n, s))).astype(np.float32)
                    for s in rank_seeds(seed, N)]
        topo = make_topo(N)
        res = two_step_allreduce_q(payloads, topo, cfg)
        rep = volume_report(res.ledger, topo)
        key = f"ts_N{N}_n{n}_b{bits}_g{g}_{'sr' if sr else 'rtn'}"
        arrays[f"in_{key}"] = np.stack(payloads)
        arrays[f"out_{key}"] = res.outputs[0]
        assert all(np.array_equal(o, res.outputs[0]) for o in res.outputs)
        index.append(dict(key=key, N=N, n=n, bits=bits, g=g, sr=sr,
                          total_raw=rep["total_raw"], total_actual=rep["total_actual"],
                          events=len(res.ledger.events)))
    # identical payloads (test_collectives.py:217-239 style)
    payload = bf16_round(gen_synthetic(default_spiky_spec(8192, 11))).astype(np.float32)
    cfg = QuantConfig(5)
    res = two_step_allreduce_q([payload.copy() for _ in range(8)], make_topo(8), cfg)
    arrays["in_ts_identical"] = payload
    arrays["out_ts_identical"] = res.outputs[0]
    index.append(dict(key="ts_identical", N=8, n=8192, bits=5, g=128, sr=False))
    arrays["index"] = np.frombuffer(json.dumps(index).encode(), dtype=np.uint8)
    np.savez_compressed(OUT / "two_step_golden.npz", **arrays)
    return len(index)


def a2a_fixture():
    arrays, index = {}, []
    N = 8
    rng = np.random.default_rng(16)
    matrix = rng.integers(0, 300, (N, N))
    matrix[2, 5] = 0
    payloads = [bf16_round(rng.normal(0, 1, int(matrix[i].sum()))).astype(np.float32)
                for i in range(N)]
    uniform = [bf16_round(gen_synthetic(default_spiky_spec(4096, s))).astype(np.float32)
               for s in rank_seeds(17, N)]
    tok = 7168 // 28  # 256-wide "tokens" keep the fixture small
    tmatrix = rng.integers(0, 6, (N, N)) * tok
    tpayloads = [bf16_round(gen_synthetic(default_spiky_spec(int(tmatrix[i].sum()) or 8, 100 + i)))
                 .astype(np.float32)[: int(tmatrix[i].sum())] for i in range(N)]
    cases = [
        ("ragged_b4_g128_sr", payloads, matrix, 4, 128, True),
        ("ragged_b6_g32_rtn", payloads, matrix, 6, 32, False),
        ("uniform_b4_g32_sr", uniform, None, 4, 32, True),
        ("tokens_b4_g128_sr", tpayloads, tmatrix, 4, 128, True),
        ("tokens_b3_g128_rtn", tpayloads, tmatrix, 3, 128, False),
    ]
    topo = preset("H800")
    for key, pl, mat, bits, g, sr in cases:
        cfg = QuantConfig(bits, group_size=g, scheme=Scheme.SPIKE_RESERVING if sr else Scheme.RTN)
        res = all2all_dispatch_q(pl, topo, cfg, mat)
        rep = volume_report(res.ledger, topo)
        for i, p in enumerate(pl):
            arrays[f"in_{key}_{i}"] = p
        if mat is not None:
            arrays[f"matrix_{key}"] = np.asarray(mat, dtype=np.int64)
        flat = np.concatenate([res.outputs[d][s] for d in range(N) for s in range(N)])
        arrays[f"out_{key}"] = flat
        index.append(dict(key=key, N=N, bits=bits, g=g, sr=sr, matrix=mat is not None,
                          total_raw=rep["total_raw"], total_actual=rep["total_actual"]))
    arrays["index"] = np.frombuffer(json.dumps(index).encode(), dtype=np.uint8)
    np.savez_compressed(OUT / "a2a_golden.npz", **arrays)
    return len(index)


def group_fixture():
    """Per-group scalar API (codec.py:278-343) and int-log scales (:366-392)."""
    from qcomm import int_to_scale, rtn_encode_group, scale_to_int, spike_encode_group

    rng = np.random.default_rng(77)
    groups = []
    for k in range(60):
        n = int(rng.integers(4, 70))
        g = rng.normal(0, 3, n)
        if k % 3 == 0:
            g[rng.integers(0, n)] *= 80.0
        if k % 7 == 0:
            g = np.round(g * 4) / 4  # exact .5 ties
        groups.append(g)
    groups += [np.full(32, 7.0), np.array([0.0, 0.5, 2.5, 3.0]), np.array([-2.0, 2.0, 0.0, 1.0]),
               np.array([100.0] + [k / 10 for k in range(1, 10)]), np.array([1.0, 1.0, 5.0, 5.0, 3.0])]
    arrays, index = {}, []
    for i, g in enumerate(groups):
        arrays[f"g{i}"] = g
        for bits in range(2, 9):
            c, s, z = rtn_encode_group(g, bits)
            arrays[f"rtn{i}_b{bits}"] = np.asarray(c, dtype=np.uint8)
            sc, m = spike_encode_group(g, bits)
            arrays[f"sr{i}_b{bits}"] = np.asarray(sc, dtype=np.uint8)
            index.append(dict(i=i, bits=bits, rtn_scale=s, rtn_zero=z, sr_scale=m.scale, sr_zero=m.zero,
                              smin=m.spike_min_value, smax=m.spike_max_value,
                              imin=m.spike_min_index, imax=m.spike_max_index))
    scales = np.concatenate([np.exp2(np.linspace(-14, 14, 2001)), [0.0, 1e-300, 1e300, 0.3, 1.0, 2.0]])
    for th in (1, 10, 37):
        arrays[f"s2i_t{th}"] = scale_to_int(scales, th)
        arrays[f"i2s_t{th}"] = int_to_scale(np.arange(-128, 128), th)
    arrays["scales"] = scales
    arrays["index"] = np.frombuffer(json.dumps(index).encode(), dtype=np.uint8)
    np.savez_compressed(OUT / "group_golden.npz", **arrays)
    return len(index)


def file_fixture():
    """FCTN -> chunk file -> FCTN through the reference CLI (cli.py:79-112)."""
    import tempfile

    from qcomm.cli import main as ref_main

    rng = np.random.default_rng(99)
    n = 3 * 4096 + 1024  # last chunk is short
    vals = (rng.normal(0, 2, n) * rng.uniform(0.01, 50, n)).astype(np.float32)
    vals[rng.integers(0, n, 40)] *= 60.0
    cases = [
        ("b5_sr_g32_bf16", ["--bitwidth", "5", "--group-size", "32", "--scheme", "sr"]),
        ("b3_rtn_g128_bf16", ["--bitwidth", "3", "--group-size", "128", "--scheme", "rtn"]),
        ("b4_sr_g128_intlog", ["--bitwidth", "4", "--group-size", "128", "--scheme", "sr",
                               "--scale-encoding", "intlog"]),
        ("b8_rtn_g64_c1024", ["--bitwidth", "8", "--group-size", "64", "--chunk-size", "1024"]),
    ]
    arrays, index = {"tensor": vals}, []
    with tempfile.TemporaryDirectory() as td:
        tin = os.path.join(td, "in.fctn")
        qcomm.fileio.write_tensor(tin, vals)
        arrays["tensor_file"] = np.frombuffer(Path(tin).read_bytes(), dtype=np.uint8)
        for key, flags in cases:
            cf, tout = os.path.join(td, key + ".fcv2"), os.path.join(td, key + ".fctn")
            assert ref_main(["quantize", "--in", tin, "--out", cf] + flags) == 0
            assert ref_main(["dequantize", "--in", cf, "--out", tout]) == 0
            arrays[f"chunks_{key}"] = np.frombuffer(Path(cf).read_bytes(), dtype=np.uint8)
            arrays[f"deq_{key}"] = np.frombuffer(Path(tout).read_bytes(), dtype=np.uint8)
            index.append(dict(key=key, flags=flags))
    arrays["index"] = np.frombuffer(json.dumps(index).encode(), dtype=np.uint8)
    np.savez_compressed(OUT / "file_golden.npz", **arrays)
    return len(index)


def hier_fixture():
    """hierarchical_two_step_q (collectives.py:318-425) on bridged fabrics:
    the 8-GPU L40 preset and a 4-GPU two-island JSON fabric."""
    four = qcomm.Topology.from_json({
        "name": "pcie4",
        "devices": [{"id": i, "sm_count": 142, "numa_group": i // 2} for i in range(4)],
        "links": [{"name": f"pcie{i}", "kind": "PCIe", "a": f"gpu{i}", "b": f"numa{i // 2}", "bandwidth": 64e9}
                  for i in range(4)] + [{"name": "bridge", "kind": "NumaBridge", "a": "numa0", "b": "numa1",
                                          "bandwidth": 32e9}]})
    cases = [
        # (topology, n, bits, g, sr, seed)
        ("L40", 16384, 4, 128, True, 20),
        ("L40", 5000, 3, 128, True, 21),
        ("L40", 8192, 2, 32, False, 22),
        ("pcie4", 3000, 5, 64, True, 23),
        ("pcie4", 4096, 8, 128, False, 24),
    ]
    arrays, index = {}, []
    for tname, n, bits, g, sr, seed in cases:
        topo = preset(tname) if tname == "L40" else four
        N = topo.n_devices
        cfg = QuantConfig(bits, group_size=g, scheme=Scheme.SPIKE_RESERVING if sr else Scheme.RTN)
        payloads = [bf16_round(gen_synthetic(default_spiky_spec(n, s))).astype(np.float32)
                    for s in rank_seeds(seed, N)]
        res = qcomm.hierarchical_two_step_q(payloads, topo, cfg)
        rep = volume_report(res.ledger, topo)
        key = f"hier_{tname}_n{n}_b{bits}_g{g}_{'sr' if sr else 'rtn'}"
        arrays[f"in_{key}"] = np.stack(payloads)
        arrays[f"out_{key}"] = np.stack(res.outputs)
        index.append(dict(key=key, topo=tname, N=N, n=n, bits=bits, g=g, sr=sr, report=rep,
                          events=[[e.stage, e.wave, e.src, e.dst, e.elements, e.actual_bytes]
                                  for e in res.ledger.events],
                          stages=[[st.name, len(st.transfers), len(st.computes)] for st in res.trace.stages]))
    arrays["index"] = np.frombuffer(json.dumps(index).encode(), dtype=np.uint8)
    arrays["topo_pcie4"] = np.frombuffer(json.dumps(four.to_json()).encode(), dtype=np.uint8)
    np.savez_compressed(OUT / "hier_golden.npz", **arrays)
    return len(index)


if __name__ == "__main__":
    if sys.argv[1:] == ["hier"]:
        print("hierarchical cases", hier_fixture())
        sys.exit(0)
    print("file cases", file_fixture())
    print("group cases", group_fixture())
    print("codec cases", codec_fixture())
    print("two-step cases", two_step_fixture())
    print("a2a cases", a2a_fixture())
