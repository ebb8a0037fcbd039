"""A/B timing of the two-step stage-2 reducer at the configs[2] shard
(8 sources x 4 Mi elements), CUDA events, L2 flushed per step.
    FC2_REDUCE=cta python tools/reduce_ab.py   # round-1 kernel"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2508_03760_b200 as fc  # noqa: E402

dev = torch.device("cuda", 0)
x = bench.spiky_bf16(8192 * 4096, 0, dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for bits, sch in ((4, "sr"), (3, "sr"), (4, "rtn"), (2, "sr"), (8, "sr")):
    cfg = fc.QuantConfig(bits, group_size=128, chunk_size=128,
                         scheme=fc.Scheme.SPIKE_RESERVING if sch == "sr" else fc.Scheme.RTN)
    r = bench.two_step_stage_times(fc, x, cfg, flush, 20)
    print(os.environ.get("FC2_REDUCE", "run"), f"b{bits}_{sch}", r["reduce_requant_8src"], flush=True)
