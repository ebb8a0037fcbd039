"""e2e host round trip vs slice size (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_03760_b200 as fc  # noqa: E402
from bench import spiky_bf16  # noqa: E402

n = 1 << 25
cfg = fc.QuantConfig(4, group_size=128, chunk_size=128, scheme=fc.Scheme.SPIKE_RESERVING)
xh = spiky_bf16(n, 0, torch.device("cuda")).cpu().pin_memory()
F = fc.footprint_bytes(cfg, n)
pay_h = torch.empty(F, dtype=torch.uint8).pin_memory()
y_h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
SL = os.environ.get("SLICES")
for sl in ([int(v) << 20 for v in SL.split(",")] if SL else [1 << 20, 1 << 21, 3 << 20, 1 << 22, 6 << 20, 1 << 23]):
    for _ in range(3):
        fc.roundtrip_host(xh, cfg, payload=pay_h, out=y_h, slice_elems=sl, check=False)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        fc.roundtrip_host(xh, cfg, payload=pay_h, out=y_h, slice_elems=sl, check=False)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"slice {sl >> 10} Ki elements: {ms:.3f} ms  {2 * n / ms / 1e6:.1f} GB/s", flush=True)
# copy floor: one H2D of x || one D2H of payload + values
xd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
pd = torch.empty(F, dtype=torch.uint8, device="cuda")
yd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    with torch.cuda.stream(s1):
        xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        pay_h.copy_(pd, non_blocking=True)
        y_h.copy_(yd, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
e.record()
torch.cuda.synchronize()
print(f"copy floor (H2D || D2H): {s.elapsed_time(e) / 5:.3f} ms", flush=True)
