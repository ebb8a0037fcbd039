"""Timeline of one fc2_roundtrip_host call at 64 MiB (dev tool; needs a
FC2_PIPE_TRACE=1 build in FC2_LIB). Prints per-slice upload / kernel /
download completion times and per-direction copy-only rates for comparison."""
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
sl = int(os.environ.get("SLICE_MI", "4")) << 20
for i in range(4):
    print(f"--- call {i}", file=sys.stderr, flush=True)
    fc.roundtrip_host(xh, cfg, payload=pay_h, out=y_h, slice_elems=sl, check=False)
torch.cuda.synchronize()
xd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
yd = torch.empty(n, dtype=torch.bfloat16, device="cuda")
for name, fn in [("H2D 64MiB alone", lambda: xd.copy_(xh, non_blocking=True)),
                 ("D2H 64MiB alone", lambda: y_h.copy_(yd, non_blocking=True))]:
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"{name}: {ms:.3f} ms = {2 * n / ms / 1e6:.1f} GB/s", file=sys.stderr, flush=True)

# control: a 4 Mi-element encode alone vs with a PCIe copy in flight on another stream
m = 4 << 20
xs_ = xd[:m]
cfg_ = cfg


def enc_time(reps=10, during=None):
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    if during is not None:
        with torch.cuda.stream(side):
            during()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fc.encode_payload(xs_, cfg_, m)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


fc.encode_payload(xs_, cfg_, m)
print(f"encode 4Mi alone: {enc_time():.1f} us/call", file=sys.stderr)
print(f"encode 4Mi during H2D: {enc_time(during=lambda: xd.copy_(xh, non_blocking=True)):.1f} us/call", file=sys.stderr)
print(f"encode 4Mi during D2H: {enc_time(during=lambda: y_h.copy_(yd, non_blocking=True)):.1f} us/call", file=sys.stderr)
print(f"encode 4Mi alone: {enc_time(reps=1):.1f} us (1 call)", file=sys.stderr)
import subprocess  # noqa: E402
import threading  # noqa: E402

clk = []


def sample():
    for _ in range(8):
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,pstate,clocks_throttle_reasons.active",
                            "--format=csv,noheader"], capture_output=True, text=True)
        clk.append(r.stdout.strip())


th = threading.Thread(target=sample)
th.start()
while th.is_alive():
    fc.roundtrip_host(xh, cfg, payload=pay_h, out=y_h, slice_elems=sl, check=False)
    torch.cuda.synchronize()
print("clocks during roundtrip_host loop:", clk, file=sys.stderr)
