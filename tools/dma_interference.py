"""Does a PCIe copy in flight slow the codec kernels? (dev tool)
Times back-to-back encodes of a 256 MiB bf16 tensor alone and while a 256 MiB
H2D / D2H copy runs on another stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_03760_b200 as fc  # noqa: E402
from bench import spiky_bf16  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 27
cfg = fc.QuantConfig(4, group_size=128, chunk_size=128, scheme=fc.Scheme.SPIKE_RESERVING)
x = spiky_bf16(n, 0, dev)
pay = fc.encode_payload(x, cfg, n)
big_h = torch.empty(1 << 28, dtype=torch.uint8).pin_memory()
big_d = torch.empty(1 << 28, dtype=torch.uint8, device=dev)
side = torch.cuda.Stream()


def run(tag, during=None, reps=8):
    torch.cuda.synchronize()
    if during is not None:
        with torch.cuda.stream(side):
            during()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fc.encode_payload(x, cfg, n, out=pay, check=False)
    e.record()
    torch.cuda.synchronize()
    print(f"{tag}: encode 256 MiB {s.elapsed_time(e) / reps * 1e3:.1f} us", flush=True)


for _ in range(2):
    run("alone")
    run("during H2D", lambda: big_d.copy_(big_h, non_blocking=True))
    run("during D2H", lambda: big_h.copy_(big_d, non_blocking=True))
    run("during both", lambda: (big_d[: 1 << 27].copy_(big_h[: 1 << 27], non_blocking=True),
                                big_h[1 << 27:].copy_(big_d[1 << 27:], non_blocking=True)))
