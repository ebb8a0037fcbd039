"""One bf16 encode + decode (b4 SR g128 by default) for ncu captures (dev tool).
KIB (default 65536 = 64 MiB), BITS, SCHEME."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_03760_b200 as fc  # noqa: E402
from bench import spiky_bf16  # noqa: E402

bits = int(os.environ.get("BITS", "4"))
sr = os.environ.get("SCHEME", "sr") == "sr"
kib = int(os.environ.get("KIB", str(64 * 1024)))
dev = torch.device("cuda", 0)
n = kib * 1024 // 2
x = spiky_bf16(n, 0, dev)
cfg = fc.QuantConfig(bits, group_size=128, chunk_size=128,
                     scheme=fc.Scheme.SPIKE_RESERVING if sr else fc.Scheme.RTN)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(2):
    flush.zero_()
    pay = fc.encode_payload(x, cfg, n)
    flush.zero_()
    y = fc.decode_payload(pay, cfg, n, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
print("ok", pay.numel(), y.numel())
