"""Event-timed encode/decode at several chunk sizes (dev tool; same flush as bench.py)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_03760_b200 as fc  # noqa: E402
from bench import flush_l2, spiky_bf16, time_roundtrip  # noqa: E402

dev = torch.device("cuda", 0)
cfg = fc.QuantConfig(4, group_size=128, scheme=fc.Scheme.SPIKE_RESERVING, chunk_size=128)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
out = {}
for m in [int(a) for a in (sys.argv[1:] or [1 << 21, 1 << 22, 3 << 21, 1 << 23, 3 << 22, 1 << 24])]:
    x = spiky_bf16(m, 3, dev)
    e, d, _, _, _ = time_roundtrip(fc, x, cfg, 10, 3, flush)
    out[m] = (round(statistics.mean(e) * 1e3, 2), round(statistics.mean(d) * 1e3, 2))
print(json.dumps(out))
