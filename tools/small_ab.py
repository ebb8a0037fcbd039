"""Back-to-back codec latency at small sizes (dev tool): region-timed like the
bench's small_message_latency.  FC2_LIB selects a library variant."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_03760_b200 as fc  # noqa: E402
from bench import spiky_bf16, time_roundtrip_region  # noqa: E402

tag = os.environ.get("TAG", "cur")
cfg = fc.QuantConfig(4, group_size=128, chunk_size=128, scheme=fc.Scheme.SPIKE_RESERVING)
x = spiky_bf16(1 << 22, 0, torch.device("cuda"))
for nb in (1 << 16, 1 << 18, 1 << 20, 1 << 22):
    m = nb // 2
    xs = [x[k * m:(k + 1) * m] for k in range(3)]
    rt, te, td, _, _ = time_roundtrip_region(fc, xs, cfg, 100, 10)
    print(f"{tag} {nb >> 10} KiB: rt {rt * 1e3:.2f} enc {te * 1e3:.2f} dec {td * 1e3:.2f} us", flush=True)
