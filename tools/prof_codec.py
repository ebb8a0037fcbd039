"""Profiling driver (dev tool): encode + decode of the bench workload a few
times, for `ncu -k regex:... --set full` captures.  Not a bench number.

    python tools/prof_codec.py [--bits 4] [--scheme sr] [--reps 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2508_03760_b200 as fc  # noqa: E402
from bench import spiky_bf16  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, default=4)
ap.add_argument("--scheme", default="sr")
ap.add_argument("--group", type=int, default=128)
ap.add_argument("--elems", type=int, default=8192 * 4096)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
torch.cuda.set_device(0)
n = a.elems
cfg = fc.QuantConfig(a.bits, group_size=a.group, chunk_size=a.group,
                     scheme=fc.Scheme.SPIKE_RESERVING if a.scheme == "sr" else fc.Scheme.RTN)
x = spiky_bf16(n, 0, torch.device("cuda", 0))
pay = torch.empty(fc.footprint_bytes(cfg, n), dtype=torch.uint8, device="cuda")
y = torch.empty(n, dtype=torch.bfloat16, device="cuda")
err = torch.zeros(1, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(a.reps):
    flush.zero_()
    fc.encode_payload(x, cfg, n, out=pay, err=err, check=False)
    flush.zero_()
    fc.decode_payload(pay, cfg, n, out=y, err=err, check=False)
torch.cuda.synchronize()
print("err", int(err.item()))

# two-step AllReduce per-rank kernels (8 shards of this tensor as 8 sources)
from bench import two_step_stage_times  # noqa: E402

two_step_stage_times(fc, x, cfg, flush, 1)
torch.cuda.synchronize()
