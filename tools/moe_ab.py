"""MoE per-rank kernel times at configs[3] (dev tool): bench.moe_stage_times."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2508_03760_b200 as fc  # noqa: E402

torch.cuda.set_device(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for bits, sch in ((4, "sr"), (4, "rtn")):
    cfg = fc.QuantConfig(bits, group_size=128, chunk_size=128,
                         scheme=fc.Scheme.SPIKE_RESERVING if sch == "sr" else fc.Scheme.RTN)
    r = bench.moe_stage_times(fc, cfg, flush, 10)
    print(os.environ.get("TAG", "cur"), f"b{bits}{sch}", json.dumps({k: v for k, v in r.items() if isinstance(v, dict)}))
