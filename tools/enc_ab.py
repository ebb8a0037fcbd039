"""A/B timing of the bf16 codec kernels (dev tool): encode-only and decode-only
regions of R back-to-back launches over 3 rotating inputs (bench.py's method),
for several sizes / bit widths, plus a payload hash (variants must match).

    FC2_LIB=variants/x/libfc2.so python tools/enc_ab.py --tag x [--reps 30] [--sizes 64,256]
"""
import argparse
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2508_03760_b200 as fc  # noqa: E402
from bench import spiky_bf16, time_roundtrip_region  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--sizes", default="16,64,256")
ap.add_argument("--cells", default="4sr,4rtn,3sr,2sr,8sr")
ap.add_argument("--tag", default="default")
a = ap.parse_args()
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
for mib in [int(v) for v in a.sizes.split(",")]:
    n = mib * (1 << 20) // 2
    xs = [spiky_bf16(n, k, dev) for k in range(3)]
    for cell in a.cells.split(","):
        bits, sch = int(cell[0]), cell[1:]
        cfg = fc.QuantConfig(bits, group_size=128, chunk_size=128,
                             scheme=fc.Scheme.SPIKE_RESERVING if sch == "sr" else fc.Scheme.RTN)
        rt, te, td, F, _ = time_roundtrip_region(fc, xs, cfg, a.reps, 3)
        pay = fc.encode_payload(xs[0], cfg, n)
        h = hashlib.sha256(pay.cpu().numpy().tobytes()).hexdigest()[:12]
        print(f"{a.tag} {mib}MiB b{bits}{sch}: enc {te * 1e3:.2f} us ({(2 * n + F) / te / 1e6:.0f} GB/s)  "
              f"dec {td * 1e3:.2f} us  rt {rt * 1e3:.2f} us  sha {h}", flush=True)
