"""Tensor / chunk files and the CLI (reference: fileio.py, cli.py:79-127).

CPU tests pin the file framing against the reference CLI's own files
(tests/golden/file_golden.npz) and the oracle; the GPU tests run the batched
quantize / dequantize and the CLI end to end and compare bytes with the
reference's files.
"""

import numpy as np
import pytest

import paper_2508_03760_b200 as fc
from oracle import fc2_oracle as O
from paper_2508_03760_b200 import fileio
from paper_2508_03760_b200.cli import main
from tests.golden_io import load

FILES, FILE_IDX = load("file_golden.npz")
IDS = [c["key"] for c in FILE_IDX]


def _flag(flags, name, default=None):
    return flags[flags.index(name) + 1] if name in flags else default


def _cfg(flags, chunk):
    return dict(bits=int(_flag(flags, "--bitwidth")), g=int(_flag(flags, "--group-size")),
                sr=_flag(flags, "--scheme", "rtn") == "sr", intlog=_flag(flags, "--scale-encoding", "bf16") == "intlog",
                chunk=int(_flag(flags, "--chunk-size", chunk)))


def test_read_tensor_matches_reference_file(tmp_path):
    p = tmp_path / "t.fctn"
    p.write_bytes(FILES["tensor_file"].tobytes())
    np.testing.assert_array_equal(fileio.read_tensor(p), FILES["tensor"])
    q = tmp_path / "u.fctn"
    fileio.write_tensor(q, FILES["tensor"])
    assert q.read_bytes() == FILES["tensor_file"].tobytes()


@pytest.mark.parametrize("bad", [b"FC", b"XXXX\x01\x00\x00\x00\x00\x00\x00\x00", b"FCTN\x02\x00\x00\x00\x00\x00\x00\x00"])
def test_read_tensor_errors(tmp_path, bad):
    p = tmp_path / "bad.fctn"
    p.write_bytes(bad)
    with pytest.raises(fc.DecodeFormatError):
        fileio.read_tensor(p)


@pytest.mark.parametrize("case", FILE_IDX, ids=IDS)
def test_chunk_file_roundtrip_and_oracle(tmp_path, case):
    """Parse the reference's chunk file, re-serialize byte-identically, and
    check every chunk against the oracle encode of its slice."""
    raw = FILES[f"chunks_{case['key']}"].tobytes()
    p = tmp_path / "c.fcv2"
    p.write_bytes(raw)
    chunks = fileio.read_chunks(p)
    q = tmp_path / "d.fcv2"
    fileio.write_chunks(q, chunks)
    assert q.read_bytes() == raw
    c = _cfg(case["flags"], 4096)
    vals = FILES["tensor"]
    pos = 0
    for ch in chunks:
        n = ch.element_count
        assert n == min(c["chunk"], vals.size - pos)
        planes, meta = O.encode(vals[pos:pos + n], c["bits"], c["g"], c["sr"], c["intlog"])
        assert ch.planes == planes and ch.meta == meta
        pos += n
    assert pos == vals.size


def test_chunk_file_truncated(tmp_path):
    raw = FILES[f"chunks_{IDS[0]}"].tobytes()
    p = tmp_path / "c.fcv2"
    p.write_bytes(raw[:-5])
    with pytest.raises(fc.DecodeFormatError):
        fileio.read_chunks(p)
    assert main(["dequantize", "--in", str(p), "--out", str(tmp_path / "o.fctn")]) == 2


def test_cli_footprint(capsys):
    assert main(["footprint", "--bitwidth", "4", "--scheme", "sr", "--group-size", "128", "--elements", "4096"]) == 0
    out = capsys.readouterr().out.strip().splitlines()
    row = dict(zip(out[0].split(","), out[1].split(",")))
    assert int(row["total"]) == O.footprint(4, 128, True, False, 4096) == 2432


def test_cli_config_error_exit_2(tmp_path):
    p = tmp_path / "t.fctn"
    p.write_bytes(FILES["tensor_file"].tobytes())
    assert main(["footprint", "--bitwidth", "9", "--elements", "4096"]) == 2


# ---------------------------------------------------------------------------
# GPU: batched quantize / dequantize == the reference CLI's files
# ---------------------------------------------------------------------------


@pytest.mark.gpu
@pytest.mark.parametrize("case", FILE_IDX, ids=IDS)
def test_gpu_cli_files_match_reference(tmp_path, case):
    tin = tmp_path / "in.fctn"
    tin.write_bytes(FILES["tensor_file"].tobytes())
    cf, tout = tmp_path / "c.fcv2", tmp_path / "o.fctn"
    assert main(["quantize", "--in", str(tin), "--out", str(cf)] + case["flags"]) == 0
    assert cf.read_bytes() == FILES[f"chunks_{case['key']}"].tobytes()
    assert main(["dequantize", "--in", str(cf), "--out", str(tout)]) == 0
    assert tout.read_bytes() == FILES[f"deq_{case['key']}"].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("case", FILE_IDX, ids=IDS)
def test_gpu_quantize_tensor_device_payload(case):
    import torch

    c = _cfg(case["flags"], 4096)
    cfg = fc.QuantConfig(c["bits"], group_size=c["g"], scheme=fc.Scheme.SPIKE_RESERVING if c["sr"] else fc.Scheme.RTN,
                         scale_encoding=fc.ScaleEncoding.INT_LOG if c["intlog"] else fc.ScaleEncoding.BF16,
                         chunk_size=c["chunk"])
    x = torch.from_numpy(FILES["tensor"]).cuda()
    chunks = fileio.quantize_tensor(x, cfg, device_payload=True)
    assert all(ch.on_device for ch in chunks)
    blob = b"".join(ch.to_bytes() for ch in chunks)
    assert blob == FILES[f"chunks_{case['key']}"].tobytes()
    y = fileio.dequantize_chunks(chunks, out_dtype=torch.float32)
    want = np.frombuffer(FILES[f"deq_{case['key']}"].tobytes()[8:], dtype="<f4")
    np.testing.assert_array_equal(y.cpu().numpy(), want)


@pytest.mark.gpu
def test_gpu_quantize_errors():
    cfg = fc.QuantConfig(4, group_size=128, chunk_size=4096)
    with pytest.raises(fc.DataError):
        fileio.quantize_tensor(np.ones(100, np.float32), cfg)
    bad = np.ones(4096, np.float32)
    bad[7] = np.inf
    with pytest.raises(fc.DataError):
        fileio.quantize_tensor(bad, cfg)


@pytest.mark.gpu
def test_gpu_cli_simulate(capsys):
    assert main(["simulate-allreduce", "--topology", "B200", "--elements", "8192", "--bitwidth", "4",
                 "--scheme", "sr", "--group-size", "128"]) == 0
    out = capsys.readouterr().out.strip().splitlines()
    row = dict(zip(out[0].split(","), out[1].split(",")))
    assert float(row["max_err"]) < 30.0
    assert main(["simulate-allreduce", "--algo", "ring", "--bitwidth", "4"]) == 2
    assert main(["simulate-all2all", "--topology", "B200", "--elements", "8192", "--bitwidth", "4"]) == 0

