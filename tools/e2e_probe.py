"""PCIe probe (dev tool): H2D / D2H alone and concurrently, and roundtrip_host
at several slice sizes, for the bench's 64 MiB bf16 chunk."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_03760_b200 as fc  # noqa: E402


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


n = 8192 * 4096
cfg = fc.QuantConfig(4, group_size=128, scheme=fc.Scheme.SPIKE_RESERVING, chunk_size=128)
F = fc.footprint_bytes(cfg, n)
xh = (torch.randn(n) * 2).to(torch.bfloat16).pin_memory()
xd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
big_h = torch.empty(n * 2 + F, dtype=torch.uint8).pin_memory()
big_d = torch.empty(n * 2 + F, dtype=torch.uint8, device="cuda")
s2 = torch.cuda.Stream()
out = {}
out["h2d_64MiB_ms"] = t(lambda: xd.copy_(xh, non_blocking=True))
out["d2h_87MB_ms"] = t(lambda: big_h.copy_(big_d, non_blocking=True))


def both():
    cur = torch.cuda.current_stream()
    s2.wait_stream(cur)
    xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        big_h.copy_(big_d, non_blocking=True)
    cur.wait_stream(s2)


out["both_concurrent_ms"] = t(both)
pay = torch.empty(F, dtype=torch.uint8).pin_memory()
y = torch.empty(n, dtype=torch.bfloat16).pin_memory()
for sl in (1 << 20, 1 << 21, 1 << 22, 1 << 23):
    out[f"roundtrip_slice_{sl >> 20}Mi_ms"] = t(lambda: fc.roundtrip_host(xh, cfg, payload=pay, out=y, slice_elems=sl,
                                                                       check=False))
print(json.dumps({k: round(v, 4) for k, v in out.items()}))
out2 = {}
for sl in (1 << 22, 1 << 23):
    out2[f"roundtrip_nopayload_slice_{sl >> 20}Mi_ms"] = t(lambda: fc.roundtrip_host(xh, cfg, payload=False, out=y,
                                                                                  slice_elems=sl, check=False))
    out2[f"encode_host_slice_{sl >> 20}Mi_ms"] = t(lambda: fc.encode_host(xh, cfg, payload=pay, slice_elems=sl,
                                                                          check=False))
    out2[f"decode_host_slice_{sl >> 20}Mi_ms"] = t(lambda: fc.decode_host(pay, cfg, n, out=y, slice_elems=sl,
                                                                          check=False))
print(json.dumps({k: round(v, 4) for k, v in out2.items()}))
